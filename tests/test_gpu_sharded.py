"""The multi-GPU (row-sharded) schedule on the device, at one rank.

A context opened with an NCCL id runs the sharded schedule even at world 1:
local rows of K.p through the non-symmetric kernels, the in-place
``ncclAllGather`` of the product slices after every matvec (engine.cpp,
lgp_api.cpp), and redundant FP64 vector updates. With one rank the gather is
an identity, so the results must equal the unsharded path's up to the kernel
choice (the unsharded CG uses the exactly symmetric K1-TC-sym). This is the
device-side coverage of the NCCL calls a one-GPU box allows; the rank-to-rank
exchange itself is covered by tests/test_dist_gloo.py on CPU."""

import ctypes as C

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import rel_l2
from oracle import gp_oracle as O
from paper_2605_17898_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sharded_ctx():
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib().lgp_comm_unique_id(buf))
    ctx = _lib.Context(0, 0, 1, buf.raw)
    yield ctx
    ctx.close()


@pytest.mark.parametrize("expr,d", [("(scale 1.2 (rbf 0.6))", 8), ("(matern52 0.7)", 3)])
def test_sharded_schedule_one_rank(gpu_ctx, sharded_ctx, expr, d):
    rng = np.random.default_rng(11)
    n = 2500
    x = rng.random((n, d))
    b = rng.standard_normal(n)
    k = G.parse_kernel(expr)
    nodes = O.parse_tree(G.format_kernel(k))

    # matvec, single and multi-RHS, through the gather
    op_s = G.KernelOperator(k, x, 0.1, ctx=sharded_ctx)
    v = rng.standard_normal(n)
    assert rel_l2(op_s(v), O.matvec(nodes, x, 0.1, v)) <= 1e-5
    V = rng.standard_normal((n, 16))
    assert rel_l2(op_s._matvec(V), O.matvec(nodes, x, 0.1, V)) <= 1e-5

    # CG: same solution as the unsharded path (its own kernel choice)
    res_s = G.cg_solve(op_s, b, G.CgConfig(rel_tolerance=1e-8))
    res = G.cg_solve(G.KernelOperator(k, x, 0.1), b, G.CgConfig(rel_tolerance=1e-8))
    assert res_s.final_residual <= 1e-8 * np.linalg.norm(b)
    assert rel_l2(res_s.x, res.x) <= 1e-4
    assert res_s.iterations <= 1.6 * res.iterations

    # Lanczos quadratures of the lockstep probes
    z = G.probe_block(n, 8, 0)
    al_s, be_s, cnt_s = op_s.lanczos(z, 10)
    al, be, cnt = G.KernelOperator(k, x, 0.1).lanczos(z, 10)
    for c in range(8):
        q_s = G.solvers.gauss_quadrature(al_s[c, :cnt_s[c]], be_s[c, :cnt_s[c] - 1])
        q = G.solvers.gauss_quadrature(al[c, :cnt[c]], be[c, :cnt[c] - 1])
        assert abs(q_s - q) <= 1e-6 * abs(q)
