"""GPU parity of the device-resident CG / SLQ loops and of the model layer
against the reference's golden outputs. Bars (north_star): predictive mean and
log marginal likelihood within 1e-4 relative of the reference at its own
tolerance / iteration budget; CG-path variance within the reference's own
cross-path tolerance 3e-3 (test_models.py:186-192)."""

import os

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import GOLDEN, golden, rel_l2
from oracle import gp_oracle as O
from paper_2605_17898_b200 import _lib

pytestmark = pytest.mark.gpu


def small_inputs(n, d, seed):
    rng = np.random.default_rng(seed)
    return rng.random((n, d)), rng.standard_normal(n)


def test_cg_golden(gpu_ctx):
    g = golden("cg_small.npz")
    for ci in range(4):
        n, d, seed = (int(a) for a in g[f"case_{ci}"])
        x, b = small_inputs(n, d, seed)
        k = G.parse_kernel(str(g[f"tree_{ci}"]))
        tol = float(g[f"tol_{ci}"])
        op = G.KernelOperator(k, x, 0.1)
        res = G.cg_solve(op, b, G.CgConfig(rel_tolerance=tol))
        it_ref = int(g[f"it_{ci}"])
        print(f"\n[cg_small case {ci}] iterations {res.iterations} vs reference {it_ref}")
        assert abs(res.iterations - it_ref) <= max(2, 0.03 * it_ref), (res.iterations, it_ref)
        assert res.final_residual <= tol * np.linalg.norm(b) or res.iterations == min(n, 1000)
        # solution vs the reference's solution
        assert rel_l2(res.x, g[f"x_{ci}"]) <= 1e-4
        # residual against the exact FP64 operator (test_models.py:97-105 style)
        gram = O.gram(O.parse_tree(G.format_kernel(k)), x, x, same=True)
        gram.flat[:: n + 1] += 0.1
        assert np.linalg.norm(gram @ res.x - b) <= max(20 * tol, 1e-5) * np.linalg.norm(b)


def test_cg_same_iteration_budget(gpu_ctx):
    # equal, pinned iteration budgets: device and oracle after exactly k steps
    x, b = small_inputs(800, 4, 21)
    k = G.Matern52(0.5)
    nodes = O.parse_tree(G.format_kernel(k))
    # un-converged iterates amplify the ~1e-7 FP32-entry perturbation with
    # every step: a CPU emulation (FP64 CG on the FP32-rounded Gram of this
    # system, cond ~2.5e3) drifts 1.4e-7 from the FP64 iterate after 5 steps and
    # 3.0e-3 after 25 (a mere FP64 re-ordering: 2e-5); the device measures
    # 4.6e-7 / 2.7e-5 (round 2), bars ~3x that. The converged-solution bar
    # (1e-4) is checked in test_cg_golden.
    for it, bar in ((5, 1.5e-6), (25, 1e-4)):
        cfg = G.CgConfig(rel_tolerance=1e-30, max_iterations=it)
        res = G.cg_solve(G.KernelOperator(k, x, 0.1), b, cfg)
        ref = O.cg(lambda v: O.matvec(nodes, x, 0.1, v), b, 1e-30, it)
        assert res.iterations == it == ref[1]
        print(f"\n[pinned budget {it}] x relL2 {rel_l2(res.x, ref[0]):.2e}")
        assert rel_l2(res.x, ref[0]) <= bar


def test_cg_multi_rhs_and_edge_columns(gpu_ctx):
    x, _ = small_inputs(600, 3, 31)
    rng = np.random.default_rng(32)
    B = rng.standard_normal((600, 5))
    B[:, 2] = 0.0  # zero column: 0 iterations, residual 0, x = 0
    op = G.KernelOperator(G.parse_kernel("(scale 1.3 (matern32 0.6))"), x, 0.2)
    X, iters, res = op.cg(B, 1e-9, None)
    assert iters[2] == 0 and res[2] == 0.0 and not X[:, 2].any()
    for c in (0, 1, 3, 4):
        one = G.cg_solve(op, np.ascontiguousarray(B[:, c]), G.CgConfig(rel_tolerance=1e-9))
        assert abs(int(iters[c]) - one.iterations) <= 1
        # the single solve runs on the symmetric tensor-core kernel, the
        # 5-column one on the SIMT kernel: two FP32-entry operators 1e-7
        # apart, amplified by the conditioning (5.5e-6 seen)
        assert rel_l2(X[:, c], one.x) <= 2e-5
    # non-convergence is reported, not raised
    X, iters, res = op.cg(B[:, :1], 1e-14, 3)
    assert iters[0] == 3 and res[0] > 0


def test_slq_golden(gpu_ctx):
    g = golden("slq_small.npz")
    for ci in range(2):
        n, d, seed, probes, steps, pseed = (int(a) for a in g[f"case_{ci}"])
        x, _ = small_inputs(n, d, seed)
        k = G.parse_kernel(str(g[f"tree_{ci}"]))
        op = G.KernelOperator(k, x, 0.1)
        ld = G.slq_logdet(op, n, G.CgConfig(probes=probes, lanczos_steps=steps), seed=pseed)
        assert abs(ld - float(g[f"logdet_{ci}"])) <= 1e-4 * abs(float(g[f"logdet_{ci}"]))
        z = G.probe_block(n, probes, pseed)
        al, be, cnt = op.lanczos(z, min(steps, n))
        for p in range(probes):
            ra = g[f"alpha_{ci}_{p}"]
            m = min(len(ra), int(cnt[p]), 8)  # leading coefficients agree closely
            np.testing.assert_allclose(al[p, :m], ra[:m], rtol=1e-5)


def test_model_cfg1_full(gpu_ctx):
    g = golden("model_cfg1.npz")
    cfg = O.CONFIGS["cfg1"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    k = G.parse_kernel(cfg["kernel"])
    st = G.gp_fit(x, y, k, cfg["noise"], "cg")
    assert abs(st.cg_iterations - int(g["it"])) <= 3
    xs = np.linspace(0.0, 1.0, 101)[:, None]
    mean, var = G.gp_predict(st, xs)
    assert rel_l2(mean, g["mean"]) <= 1e-4
    assert np.max(np.abs(var - g["var"])) <= 3e-3
    assert np.max(np.abs(mean - g["chol_mean"])) <= 1e-4 * np.abs(g["chol_mean"]).max() + 1e-5
    lml = G.log_marginal_likelihood(st, seed=0)
    assert abs(lml - float(g["lml"])) <= 1e-4 * abs(float(g["lml"]))


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "model_small.npz")),
                    reason="model_small fixture not generated")
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_model_small_matrix_free_branch(gpu_ctx, name):
    g = golden("model_small.npz")
    cfg = O.CONFIGS[name]
    x, y = O.synthetic(3000, cfg["d"])
    xs = np.random.default_rng(9).random((8, cfg["d"]))
    st = G.gp_fit(x, y, G.parse_kernel(cfg["kernel"]), cfg["noise"], "cg")
    it_ref = int(g[f"{name}_it"])
    print(f"\n[model_small {name}] iterations {st.cg_iterations} vs reference {it_ref}")
    assert abs(st.cg_iterations - it_ref) <= max(3, 0.03 * it_ref)
    mean, var = G.gp_predict(st, xs)
    assert rel_l2(mean, g[f"{name}_mean"]) <= 1e-4
    assert np.max(np.abs(var - g[f"{name}_var"])) <= 3e-3
    lml = G.log_marginal_likelihood(st, seed=0)
    assert abs(lml - float(g[f"{name}_lml"])) <= 1e-4 * abs(float(g[f"{name}_lml"]))


def _fp64_cg(expr, x, b, tol=1e-8):
    """The reference algorithm (solvers.py:87-123) on the exact FP64 Gram."""
    nodes = O.parse_tree(expr)
    gram = O.gram(nodes, x, x, same=True)
    gram.flat[:: x.shape[0] + 1] += 0.1
    return O.cg(lambda v: gram @ v, b, tol)


@pytest.mark.parametrize("nwg,r", [("4", ""), ("3", ""), ("4", "1"), ("4", "3")])
def test_symmetric_tensor_core_cg(gpu_ctx, monkeypatch, nwg, r):
    """The symmetric tensor-core CG matvec (default for D >= 4 r^2 trees)
    evaluates each unordered pair once: exactly symmetric, so CG tracks the
    reference algorithm on the exact FP64 Gram (iterations, solution), like
    the symmetric SIMT kernel (LGP_NO_TCSYM) does, for 4 and 3 epilogue
    warpgroups and forced super-tile sizes (LGP_TS_R; default: the scheduling
    model's choice); the matvec meets the 1e-5 bar."""
    x, b = small_inputs(3000, 8, 41)
    expr = "(scale 1.2 (rbf 0.6))"
    k = G.parse_kernel(expr)
    ref = _fp64_cg(expr, x, b)
    monkeypatch.setenv("LGP_NO_TCSYM", "1")
    base = G.cg_solve(G.KernelOperator(k, x, 0.1, ctx=_lib.Context(0)), b, G.CgConfig(rel_tolerance=1e-8))
    monkeypatch.delenv("LGP_NO_TCSYM")
    monkeypatch.setenv("LGP_TS_NWG", nwg)
    if r:
        monkeypatch.setenv("LGP_TS_R", r)
    op = G.KernelOperator(k, x, 0.1, ctx=_lib.Context(0))
    res = G.cg_solve(op, b, G.CgConfig(rel_tolerance=1e-8))
    print(f"\n[tcsym nwg={nwg} R={r or 'auto'}] iterations {res.iterations}, SIMT-sym {base.iterations}, "
          f"FP64 reference {ref[1]}; x relL2 {rel_l2(res.x, ref[0]):.1e} (SIMT-sym {rel_l2(base.x, ref[0]):.1e})")
    for it, xs in ((res.iterations, res.x), (base.iterations, base.x)):
        assert abs(it - ref[1]) <= max(3, 0.05 * ref[1])
        assert rel_l2(xs, ref[0]) <= 1e-4
    v = np.random.default_rng(5).standard_normal(3000)
    want = O.matvec(O.parse_tree(expr), x, 0.1, v)
    assert rel_l2(op(v), want) <= 1e-5


def test_evidence_optimizer_matches_reference(gpu_ctx):
    """3 Adam steps of central-difference ascent on the exact-GP evidence
    (every evaluation a device CG fit + device SLQ) track the reference's own
    run (dense CG operator, SLQ seed 0) - the §8f caller of the fit path."""
    g = golden("optimizer.npz")
    rng = np.random.default_rng(17)
    x = rng.random((600, 3))
    y = np.sin(2.0 * x.sum(1)) + 0.1 * rng.standard_normal(600)
    kernel = G.parse_kernel("(scale 1.0 (rbf 0.5))")
    cfg = G.OptimizerConfig(steps=3, learning_rate=0.05)
    obj = G.exact_evidence_objective(x, y, kernel, seed=0)
    best, trace = G.optimize_hyperparams(obj, G.flatten_model_params(kernel, 0.1), cfg)
    assert cfg.evaluations == int(g["gp_evals"]) == 21
    np.testing.assert_allclose(np.array(trace), g["gp_trace"], rtol=1e-4)
    np.testing.assert_allclose(best, g["gp_best"], atol=2e-3)


@pytest.mark.parametrize("d,expr", [(4, "(matern52 0.7)"), (40, "(rbf 2.5)"),
                                    (2, "(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))")])
def test_symmetric_tensor_core_cg_dims(gpu_ctx, monkeypatch, d, expr):
    """The default CG matvec for r^2 / Periodic trees (K1-TC-sym) at the
    smallest and a large feature dimension: iterations and solution track the
    reference algorithm on the exact FP64 Gram, as the SIMT kernel's do."""
    x, b = small_inputs(2500, d, 43)
    k = G.parse_kernel(expr)
    ref = _fp64_cg(expr, x, b)
    monkeypatch.setenv("LGP_NO_TCSYM", "1")
    base = G.cg_solve(G.KernelOperator(k, x, 0.1, ctx=_lib.Context(0)), b, G.CgConfig(rel_tolerance=1e-8))
    monkeypatch.delenv("LGP_NO_TCSYM")
    res = G.cg_solve(G.KernelOperator(k, x, 0.1, ctx=_lib.Context(0)), b, G.CgConfig(rel_tolerance=1e-8))
    print(f"\n[tcsym d={d} {expr}] iterations {res.iterations}, SIMT-sym {base.iterations}, FP64 reference "
          f"{ref[1]}; x relL2 {rel_l2(res.x, ref[0]):.1e} (SIMT-sym {rel_l2(base.x, ref[0]):.1e})")
    # the RBF + Periodic system at D = 2 is the rounding-sensitive one: its
    # recurrence residual reaches 1e-8 between 170 and 184 iterations depending
    # on the summation order alone (super-tile sizes R = 1..8: 178-179; the
    # default schedule: 170; FP64: 184) while the solution error stays 2e-5
    # (tools/tcsym_repeat.py)
    bar = 0.10 if "periodic" in expr else 0.05
    for it, xs in ((res.iterations, res.x), (base.iterations, base.x)):
        assert abs(it - ref[1]) <= max(3, bar * ref[1])
        assert rel_l2(xs, ref[0]) <= 1e-4


@pytest.mark.parametrize("expr,d", [("(scale 1.2 (rbf 0.6))", 8),
                                    ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 2)])
def test_device_results_are_deterministic(gpu_ctx, expr, d):
    """Every reduction on the device runs in a fixed order (no atomics): the
    same inputs give bit-identical products, CG iterates and Lanczos
    coefficients on repeated calls (tensor-core, symmetric and SIMT paths)."""
    x, b = small_inputs(6000, d, 47)
    k = G.parse_kernel(expr)
    op = G.KernelOperator(k, x, 0.1)
    V = np.random.default_rng(3).standard_normal((6000, 16))
    m1, m2 = op(V), op(V)
    np.testing.assert_array_equal(m1, m2)
    v1, v2 = op(b), op(b)
    np.testing.assert_array_equal(v1, v2)
    r1 = G.cg_solve(op, b, G.CgConfig(rel_tolerance=1e-8))
    r2 = G.cg_solve(G.KernelOperator(k, x, 0.1), b, G.CgConfig(rel_tolerance=1e-8))
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(r1.x, r2.x)
    z = G.probe_block(6000, 16, 0)
    a1, b1, c1 = op.lanczos(z, 20)
    a2, b2, c2 = op.lanczos(z, 20)
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(b1, b2)


def test_evidence_objective_batch_matches_sequential(gpu_ctx):
    """An optimiser step's 2P + 1 evidence evaluations at once: without shift
    fusion (concurrent per-thread contexts) bit-identical to one-by-one calls;
    with it (points differing only in the output scale / noise share one
    multi-shift CG and one Lanczos run, §8f row 3) within 1e-9 relative."""
    rng = np.random.default_rng(23)
    x = rng.random((900, 3))
    y = np.sin(2.0 * x.sum(1)) + 0.1 * rng.standard_normal(900)
    kernel = G.parse_kernel("(scale 1.2 (rbf 0.4))")
    p = G.flatten_model_params(kernel, 0.1)
    qs = [p, *[p + np.eye(3)[i] * s for i in range(3) for s in (1e-4, -1e-4)]]
    seq = [G.exact_evidence_objective(x, y, kernel, seed=0)(q) for q in qs]
    plain = G.exact_evidence_objective(x, y, kernel, seed=0, workers=7, fuse_shifts=False)
    assert plain.batch(qs) == seq
    fused = G.exact_evidence_objective(x, y, kernel, seed=0, workers=3).batch(qs)
    err = max(abs(a - b) / abs(b) for a, b in zip(fused, seq))
    print(f"\n[fused 2P+1 batch] max relative difference to sequential {err:.1e}")
    assert err <= 1e-9


@pytest.mark.parametrize("seed,n,d", [(0, 300, 2), (1, 1000, 2), (2, 3000, 8)])
def test_cg_gram_operators_match_cholesky(gpu_ctx, seed, n, d):
    """Reference test_solvers.py:133-147 on the device operator: CG at tol 1e-11
    against an FP64 Cholesky solve of the same Gram. The reference's 1e-8
    bar is for FP64 entries; with FP32 entries the solutions agree to
    ~1e-6 relative (3e-6 absolute measured), bar 1e-5 relative."""
    import scipy.linalg

    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    y = rng.standard_normal(n)
    k = G.Scale(1.3, G.RBF(0.3))
    gram = O.gram(O.parse_tree(G.format_kernel(k)), x, x, same=True)
    gram.flat[:: n + 1] += 1.0
    want = scipy.linalg.cho_solve(scipy.linalg.cho_factor(gram), y)
    res = G.cg_solve(G.KernelOperator(k, x, 1.0), y,
                     G.CgConfig(rel_tolerance=1e-11, max_iterations=5 * n))
    assert rel_l2(res.x, want) <= 1e-5
    assert np.max(np.abs(res.x - want)) <= 3e-5


def test_multi_rhs_cg_column_compaction(gpu_ctx, monkeypatch):
    """The multi-RHS CG (predictive variance) drops converged columns from its
    K1 passes: same per-column iterations, residuals and solutions as keeping
    every column (LGP_CG_NO_COMPACT=1). 130 columns = 3 passes of 64; three
    zero columns finish at once (0 iterations) so the rest fit 2 passes from
    the first check on, and smooth k* columns converge apart from random
    ones."""
    x, _ = small_inputs(4000, 8, 61)
    rng = np.random.default_rng(62)
    B = rng.standard_normal((4000, 130))
    B[:, ::7] = G.kernel_eval(G.parse_kernel("(rbf 0.5)"), x, rng.random((19, 8)))
    B[:, [5, 50, 100]] = 0.0
    k = G.parse_kernel("(rbf 0.5)")
    op = G.KernelOperator(k, x, 0.1)
    X1, it1, r1 = op.cg(B, 1e-8, None)
    monkeypatch.setenv("LGP_CG_NO_COMPACT", "1")
    X0, it0, r0 = op.cg(B, 1e-8, None)
    print(f"\n[compaction] iterations min/max {it1.min()}/{it1.max()}")
    assert it1.max() > it1.min() + 8  # columns really converge at different iterations
    np.testing.assert_array_equal(it1, it0)
    np.testing.assert_array_equal(r1, r0)
    np.testing.assert_array_equal(X1, X0)


@pytest.mark.parametrize("expr,d", [("(rbf 0.5)", 8), ("(matern52 0.7)", 3)])
def test_multi_shift_cg_matches_separate_solves(gpu_ctx, expr, d):
    """lgp_cg_shifted (one matvec per iteration for every shift: CG-M)
    reproduces separate CG solves of (K + (noise + shift) I) x = b. The
    optimiser's shifts are small (finite-difference steps of the noise and the
    output scale): iteration counts within rounding noise of the stop rule
    (+-3: the separate solves themselves move that much with the noise value's
    rounding) and solutions to 1e-6, the seed itself bit for bit. Large shifts converge much faster than the seed, and
    their residual, read off the seed's recurrence (|zeta| ||r||), is then
    less accurate: iterations within 5 %."""
    x, b = small_inputs(3000, d, 71)
    k = G.parse_kernel(expr)
    noise = 0.05
    shifts = np.array([0.0, 1e-4, 1e-3, 0.01, 0.05, 0.3, 1.7])
    op = G.KernelOperator(k, x, noise)
    X, it, res = op.cg_shifted(b, shifts, 1e-8, None)
    for e, sh in enumerate(shifts):
        one = G.cg_solve(G.KernelOperator(k, x, noise + sh), b, G.CgConfig(rel_tolerance=1e-8))
        err = rel_l2(X[:, e], one.x)
        print(f"\n[shift {sh}] iterations {it[e]} vs {one.iterations}, x relL2 {err:.1e}, "
              f"residual {res[e]:.2e} vs {one.final_residual:.2e}")
        assert res[e] <= 1e-8 * np.linalg.norm(b)
        if sh <= 0.05:
            assert abs(int(it[e]) - one.iterations) <= 3
            assert err <= 1e-6
        else:
            assert abs(int(it[e]) - one.iterations) <= max(2, 0.05 * one.iterations)
            assert err <= 1e-5
        if sh == 0.0:
            assert int(it[e]) == one.iterations
            np.testing.assert_array_equal(X[:, e], one.x)


@pytest.mark.parametrize("expr,d,n,noise", [("(scale 1.3 (rbf 0.5))", 8, 9000, 0.1),
                                            ("(+ (scale 1.0 (rbf 0.5)) (scale 0.5 (periodic 1.0 0.8)))", 2, 7000, 0.05)])
def test_one_launch_cg_vector_step_is_bit_identical(gpu_ctx, monkeypatch, expr, d, n, noise):
    """The cooperative one-launch vector step (k_cg1_vec) reproduces the
    three-kernel step (records + p.Ap + step | x/r update + r.r + beta | next
    direction) bit for bit: same shares, same fixed summation orders."""
    rng = np.random.default_rng(11)
    x, b = rng.random((n, d)), rng.standard_normal(n)
    op = G.KernelOperator(G.parse_kernel(expr), x, noise)
    x1, it1, r1 = op.cg(b, 1e-9, None)
    x1, it1, r1 = x1.copy(), int(it1[0]), float(r1[0])
    monkeypatch.setenv("LGP_CG_VEC3", "1")
    x3, it3, r3 = op.cg(b, 1e-9, None)
    assert it1 == int(it3[0]) and r1 == float(r3[0])
    np.testing.assert_array_equal(x1, x3)
