"""Device-side error semantics of the solver loops (reference solvers.py):

* CG breakdown p.A.p <= 0 -> OperatorNotSpdError (solvers.py:110-113;
  reference test pkg/tests/test_solvers.py:160, `cg_solve(lambda v: -v, ...)`),
  raised from lgp_cg's device finalize - on the symmetric tensor-core kernel
  (fused iteration) and on the SIMT kernels;
* a nonpositive Ritz value of the Lanczos tridiagonal -> OperatorNotSpdError
  (solvers.py:156-159; reference test pkg/tests/test_solvers.py:214) from the
  device Lanczos's coefficients;
* the solver state is usable afterwards (the next call on the same context
  solves normally).

Kernel operators are PSD by construction, so the non-SPD operators here are
singular ones whose products are exactly zero: the Linear kernel on zero
points (K = 0) with noise 0, and RBF on identical points (K = kappa 1 1^T,
every entry the same FP32 number) applied to a +-1 vector summing to 0.
"""

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from paper_2605_17898_b200.errors import OperatorNotSpdError

pytestmark = pytest.mark.gpu


def test_cg_breakdown_simt_kernel(gpu_ctx):
    x = np.zeros((300, 3))
    op = G.KernelOperator(G.parse_kernel("(linear 1.0)"), x, 0.0)
    with pytest.raises(OperatorNotSpdError):
        G.cg_solve(op, np.ones(300), G.CgConfig())


def test_cg_breakdown_symmetric_tensor_core_kernel(gpu_ctx):
    # identical points: every entry is the same FP32 value; b sums to zero, so
    # K b = 0 exactly and p.A.p = 0 at the first iteration
    n = 4096
    x = np.full((n, 8), 0.3)
    b = np.tile([1.0, -1.0], n // 2)
    op = G.KernelOperator(G.parse_kernel("(rbf 0.5)"), x, 0.0)
    assert "lgp_matvec_tcsym" in G.kernels.program(op.kernel).source(8, 16)
    with pytest.raises(OperatorNotSpdError):
        G.cg_solve(op, b, G.CgConfig())
    # the context keeps working: a regular solve right after the breakdown
    rng = np.random.default_rng(1)
    x2 = rng.random((n, 8))
    op2 = G.KernelOperator(G.parse_kernel("(rbf 0.5)"), x2, 0.1)
    res = G.cg_solve(op2, rng.standard_normal(n), G.CgConfig(rel_tolerance=1e-8))
    assert res.final_residual > 0 and res.iterations > 1


def test_cg_breakdown_multi_rhs(gpu_ctx):
    # multi-RHS device CG (predictive variance path): a zero column among
    # regular ones still breaks down on the zero operator
    x = np.zeros((200, 2))
    op = G.KernelOperator(G.parse_kernel("(linear 0.7)"), x, 0.0)
    with pytest.raises(OperatorNotSpdError):
        op.cg(np.ones((200, 3)), 1e-8, None)


def test_lanczos_nonpositive_ritz_value(gpu_ctx):
    x = np.zeros((64, 2))
    op = G.KernelOperator(G.parse_kernel("(linear 1.0)"), x, 0.0)
    with pytest.raises(OperatorNotSpdError):
        G.slq_logdet(op, 64, G.CgConfig(probes=2, lanczos_steps=8), seed=0)


def test_lanczos_nonpositive_ritz_value_tensor_core(gpu_ctx):
    # K = kappa 1 1^T, noise 0: the Krylov space of a probe is span{z, 1}, the
    # tridiagonal's smallest Ritz value is 0 up to rounding (<= 0 raises; a
    # positive rounding residue is what the reference would see too, so the
    # zero operator above is the exact case) - here only the call must not
    # hang or return NaN
    n = 2048
    x = np.full((n, 8), 0.25)
    op = G.KernelOperator(G.parse_kernel("(rbf 0.5)"), x, 0.0)
    try:
        ld = G.slq_logdet(op, n, G.CgConfig(probes=4, lanczos_steps=10), seed=0)
        assert np.isfinite(ld)
    except OperatorNotSpdError:
        pass
