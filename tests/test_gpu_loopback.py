"""Multi-rank engine bookkeeping on one GPU (TEST-ONLY loopback group).

G ranks of one process, each with its own library context on the same GPU,
driven by host threads; the library's all-gather is host-mediated for a
"LGP-LOOPBACK" id (stream sync, host barrier, device-to-device copies: no
kernel waits on another rank, so nothing relies on co-scheduling). This runs
the real multi-rank code of lgp_matvec / lgp_cg / lgp_lanczos — row
partitions, padded last slices (n not divisible by G), row offsets, the
in-place gather — and checks that every rank ends with identical state equal
to the one-rank result. The NCCL transport itself is exercised at one rank by
tests/test_gpu_sharded.py and across processes (CPU, gloo) by
tests/test_dist_gloo.py."""

import os
import threading

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import rel_l2
from oracle import gp_oracle as O
from paper_2605_17898_b200 import _lib

pytestmark = pytest.mark.gpu


def run_ranks(world, fn):
    gid = b"LGP-LOOPBACK" + os.urandom(16)
    gid = gid + bytes(128 - len(gid))
    out, errs = [None] * world, []

    def worker(r):
        try:
            ctx = _lib.Context(0, r, world, gid)
            try:
                out[r] = fn(ctx, r)
            finally:
                ctx.close()
        except Exception as exc:  # reported below
            errs.append((r, repr(exc)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_ranks_match_one_rank(gpu_ctx, world):
    rng = np.random.default_rng(5)
    n, d = 2051, 5  # n % world != 0: padded last slice
    x = rng.random((n, d))
    b = rng.standard_normal(n)
    V = rng.standard_normal((n, 16))
    k = G.parse_kernel("(+ (scale 1.1 (rbf 0.6)) (scale 0.4 (matern32 0.9)))")
    nodes = O.parse_tree(G.format_kernel(k))
    z = G.probe_block(n, 8, 0)

    def fn(ctx, r):
        op = G.KernelOperator(k, x, 0.1, ctx=ctx)
        mv = op._matvec(V).copy()
        xs, it, res = op.cg(b, 1e-8, None)
        al, be, cnt = op.lanczos(z, 12)
        return mv, xs.copy(), int(it[0]), float(res[0]), al.copy(), cnt.copy(), be.copy()

    outs = run_ranks(world, fn)
    ref = run_ranks(1, fn)[0]  # one rank, same (sharded) schedule
    for r in range(world):
        mv, xs, it, res, al, cnt, be = outs[r]
        # every rank holds the full product / iterates, identical across ranks
        np.testing.assert_array_equal(mv, outs[0][0])
        np.testing.assert_array_equal(xs, outs[0][1])
        assert it == outs[0][2]
        np.testing.assert_array_equal(al, outs[0][4])
    mv, xs, it, res, al, cnt, be = outs[0]
    assert rel_l2(mv, O.matvec(nodes, x, 0.1, V)) <= 1e-5
    assert rel_l2(mv, ref[0]) <= 1e-6
    assert abs(it - ref[2]) <= max(2, 0.03 * ref[2])
    assert res <= 1e-8 * np.linalg.norm(b)
    assert rel_l2(xs, ref[1]) <= 1e-5
    np.testing.assert_array_equal(cnt, ref[5])
    # late Lanczos coefficients amplify rounding-order differences of the
    # matvec (1.5e-5 seen at step 12); the quadratures they feed are stable
    np.testing.assert_allclose(al[:, :4], ref[4][:, :4], rtol=3e-6)  # 1.3e-6 seen
    for c in range(8):
        m = int(cnt[c])
        q = G.solvers.gauss_quadrature(al[c, :m], be[c, :m - 1])
        q1 = G.solvers.gauss_quadrature(ref[4][c, :m], ref[6][c, :m - 1])
        assert abs(q - q1) <= 1e-5 * abs(q1), (c, q, q1)  # 2.7e-7 seen


def test_loopback_more_ranks_than_work(gpu_ctx):
    """world 4 on a 300-point operator: some ranks own no pair items of the
    symmetric CG (empty launch, no records) and the row slices are tiny; every
    rank still ends with the one-rank solution."""
    rng = np.random.default_rng(9)
    n, d = 300, 5
    x = rng.random((n, d))
    b = rng.standard_normal(n)
    k = G.parse_kernel("(scale 1.3 (rbf 0.7))")

    def fn(ctx, r):
        op = G.KernelOperator(k, x, 0.1, ctx=ctx)
        xs, it, res = op.cg(b, 1e-8, None)
        return xs.copy(), int(it[0]), op._matvec(np.ascontiguousarray(
            np.random.default_rng(2).standard_normal((n, 9)))).copy()

    outs = run_ranks(4, fn)
    ref = run_ranks(1, fn)[0]
    for r in range(4):
        np.testing.assert_array_equal(outs[r][0], outs[0][0])
        assert outs[r][1] == outs[0][1]
        np.testing.assert_array_equal(outs[r][2], outs[0][2])
    assert abs(outs[0][1] - ref[1]) <= 2
    assert rel_l2(outs[0][0], ref[0]) <= 1e-6
    assert rel_l2(outs[0][2], ref[2]) <= 1e-6
