"""Full-size ("tier C") parity against the real reference.

* cfg2 in full (N = 20000, Matern-5/2, D = 4): gp_fit (CG, tol 1e-8) /
  gp_predict / log_marginal_likelihood against the reference's own CG / SLQ
  code on the dense-replay operator (tests/golden/make_tierc.py). Bars: the
  north star's (mean and LML 1e-4 relative; variance 3e-3 absolute against the
  exact Cholesky variance; iteration count within 10 %).
* cfg4 (N = 100000, RBF, D = 8) at equal, pinned budgets through the reference's
  real matrix_free_matvec: CG after exactly 20 iterations and the Lanczos
  quadratures of 16 probes after 5 steps.
* the cfg4 kernel (RBF 0.5, D = 8) and the cfg5 kernel (Matern-3/2 0.5, D = 8)
  CONVERGED at N = 50000 (the largest N whose FP64 dense replay fits the build
  container, SURVEY.md §8c tier C): gp_fit (CG, tol 1e-8) / gp_predict (200
  test points) / log_marginal_likelihood against the reference's own
  cg_solve / slq_logdet on the dense replay, variance against the exact
  (Cholesky) one. Bars (north star): iterations within 3 %, alpha / mean / LML
  within 1e-4 relative, variance within 3e-3 absolute.
"""

import os

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import GOLDEN, golden, rel_l2
from oracle import gp_oracle as O

pytestmark = pytest.mark.gpu

# ~3x the measured errors of the pinned 20-iteration cfg4 CG (round 2 on the
# B200: x relL2 9.4e-7, final residual 4.9e-8 relative)
TIERC_CFG4_X_BAR = 3e-6
TIERC_CFG4_RES_BAR = 1.5e-7


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "fullsize_cfg2.npz")),
                    reason="fullsize_cfg2 fixture not generated")
def test_fullsize_cfg2_fit_predict_lml(gpu_ctx):
    g = golden("fullsize_cfg2.npz")
    cfg = O.CONFIGS["cfg2"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    st = G.gp_fit(x, y, G.parse_kernel(cfg["kernel"]), cfg["noise"], "cg")
    it_ref = int(g["it"])
    print(f"\n[fullsize cfg2] iterations {st.cg_iterations} vs reference {it_ref}")
    assert abs(st.cg_iterations - it_ref) <= max(3, 0.03 * it_ref), (st.cg_iterations, it_ref)
    assert rel_l2(st.alpha, g["alpha"]) <= 1e-4
    xs = np.random.default_rng(9).random((200, cfg["d"]))
    mean, var = G.gp_predict(st, xs)
    assert rel_l2(mean, g["mean"]) <= 1e-4
    assert np.max(np.abs(var - g["var"])) <= 3e-3
    lml = G.log_marginal_likelihood(st, seed=0)
    assert abs(lml - float(g["lml"])) <= 1e-4 * abs(float(g["lml"])), (lml, float(g["lml"]))


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "tierc_cfg4.npz")),
                    reason="tierc_cfg4 fixture not generated")
def test_tierc_cfg4_pinned_budgets(gpu_ctx):
    g = golden("tierc_cfg4.npz")
    cfg = O.CONFIGS["cfg4"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"])
    res = G.cg_solve(op, y, G.CgConfig(rel_tolerance=1e-30, max_iterations=int(g["it"])))
    assert res.iterations == int(g["it"])
    # un-converged iterates carry the FP32-entry perturbation amplified by the
    # iteration; the bars are 3x the measured values (printed)
    e_x = rel_l2(res.x, g["x"])
    e_r = abs(res.final_residual - float(g["res"])) / float(g["res"])
    print(f"\n[tier C cfg4, 20 pinned CG iterations] x relL2 {e_x:.2e}, residual rel {e_r:.2e}")
    assert e_x <= TIERC_CFG4_X_BAR
    assert e_r <= TIERC_CFG4_RES_BAR
    steps, probes = int(g["steps"]), int(g["probes"])
    z = G.probe_block(cfg["n"], probes, 0)
    al, be, cnt = op.lanczos(z, steps)
    for c in range(probes):
        m = int(cnt[c])
        q = G.solvers.gauss_quadrature(al[c, :m], be[c, :m - 1])
        assert abs(q - g["quads"][c]) <= 1e-5 * abs(g["quads"][c]), (c, q, g["quads"][c])


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "tierc_cfg3.npz")),
                    reason="tierc_cfg3 fixture not generated")
def test_tierc_cfg3_pinned_budgets(gpu_ctx):
    """cfg3 (RBF + Periodic, N = 50000, D = 2: the Periodic features ride next
    to the tensor-core distance tile) through the reference's real
    matrix_free_matvec: CG after exactly 10 iterations, the Lanczos
    quadratures of 4 probes after 3 steps."""
    g = golden("tierc_cfg3.npz")
    cfg = O.CONFIGS["cfg3"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"])
    res = G.cg_solve(op, y, G.CgConfig(rel_tolerance=1e-30, max_iterations=int(g["it"])))
    assert res.iterations == int(g["it"])
    # measured 3e-7 / 1.4e-8 / <= 2.7e-7 (tools/tierc3_check.py)
    assert rel_l2(res.x, g["x"]) <= 1e-5
    assert abs(res.final_residual - float(g["res"])) <= 1e-5 * float(g["res"])
    steps, probes = int(g["steps"]), int(g["probes"])
    z = G.probe_block(cfg["n"], probes, 0)
    al, be, cnt = op.lanczos(z, steps)
    for c in range(probes):
        m = int(cnt[c])
        q = G.solvers.gauss_quadrature(al[c, :m], be[c, :m - 1])
        assert abs(q - g["quads"][c]) <= 1e-5 * abs(g["quads"][c]), (c, q, g["quads"][c])


@pytest.mark.parametrize("tag", ["rbf", "m32"])
def test_tierc_n50k_converged_fit_predict_lml(gpu_ctx, tag):
    path = os.path.join(GOLDEN, f"tierc_n50k_{tag}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = golden(f"tierc_n50k_{tag}.npz")
    n, d, noise = int(g["n"]), int(g["d"]), float(g["noise"])
    x, y = O.synthetic(n, d)
    st = G.gp_fit(x, y, G.parse_kernel(str(g["kernel"])), noise, "cg")
    it_ref = int(g["it"])
    e_alpha = rel_l2(st.alpha, g["alpha"])
    xs = np.random.default_rng(9).random((200, d))
    mean, var = G.gp_predict(st, xs)
    e_mean = rel_l2(mean, g["mean"])
    e_var = float(np.max(np.abs(var - g["var"])))
    lml = G.log_marginal_likelihood(st, seed=0)
    e_lml = abs(lml - float(g["lml"])) / abs(float(g["lml"]))
    print(f"\n[tier C n50k {tag}] iterations {st.cg_iterations} vs reference {it_ref}; "
          f"alpha relL2 {e_alpha:.2e}, mean relL2 {e_mean:.2e}, var max abs {e_var:.2e}, "
          f"LML rel {e_lml:.2e}")
    assert abs(st.cg_iterations - it_ref) <= 0.03 * it_ref, (st.cg_iterations, it_ref)
    assert e_alpha <= 1e-4
    assert e_mean <= 1e-4
    assert e_var <= 3e-3
    assert e_lml <= 1e-4, (lml, float(g["lml"]))
