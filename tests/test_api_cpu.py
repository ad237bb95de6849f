"""Host-side API surface (no GPU): kernel algebra, hyper-parameter interface,
grammar, lowering, argument validation, and the generic-callable CG / SLQ
contract — mirroring the reference's own unit tests (pkg/tests/test_kernels.py,
test_solvers.py)."""

import math

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import golden
from paper_2605_17898_b200 import kernels as K


def test_kernel_validation_and_sugar():
    with pytest.raises(ValueError):
        G.RBF(0.0)
    with pytest.raises(ValueError):
        G.Periodic(1.0, -2.0)
    with pytest.raises(ValueError):
        G.Scale(float("nan"), G.RBF())
    with pytest.raises(TypeError):
        G.Scale(1.0, 3)
    with pytest.raises(TypeError):
        G.Sum(G.RBF(), "x")
    k = G.RBF(0.5) + G.Scale(2.0, G.Periodic(1.0, 0.5)) * G.Linear(0.3)
    assert isinstance(k, G.Sum) and isinstance(k.right, G.Product)
    with pytest.raises(Exception):
        k.left.lengthscale = 3.0  # frozen


def test_params_roundtrip_preorder():
    k = G.Sum(G.Scale(1.5, G.Matern32(0.4)), G.Product(G.Periodic(0.8, 1.3), G.Linear(0.2)))
    assert k._params() == (1.5, 0.4, 0.8, 1.3, 0.2)
    assert G.n_params(k) == 5
    v = G.flatten_params(k)
    np.testing.assert_allclose(v, np.log([1.5, 0.4, 0.8, 1.3, 0.2]))
    k2 = G.unflatten_params(k, v)
    assert k2 == k or np.allclose(k2._params(), k._params())
    with pytest.raises(G.DimensionMismatchError):
        G.unflatten_params(k, v[:3])
    with pytest.raises(G.NonFiniteError):
        G.unflatten_params(k, np.array([0, 0, np.nan, 0, 0.0]))


@pytest.mark.parametrize("text", [
    "(rbf 0.5)", "(matern12 0.3)", "(matern32 0.4)", "(matern52 0.5)", "(periodic 0.8 1.3)",
    "(linear 0.7)", "(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))",
    "(* (scale 0.7 (matern52 0.9)) (+ (matern12 1.1) (rbf 0.3)))",
])
def test_grammar_roundtrip(text):
    k = G.parse_kernel(text)
    assert G.parse_kernel(G.format_kernel(k)) == k


@pytest.mark.parametrize("bad,token", [
    ("", None), ("rbf 0.5", "rbf"), ("(rbf)", ")"), ("(rbf x)", "x"), ("(foo 1)", "foo"),
    ("(rbf 0.5) (rbf 1)", "("), ("(rbf -1)", "rbf"), ("(rbf 0.5", None),
])
def test_grammar_errors(bad, token):
    with pytest.raises(G.KernelParseError) as e:
        G.parse_kernel(bad)
    if token is not None:
        assert e.value.token == token


def test_slab_buffers_and_stationary():
    assert G.slab_buffer_count(G.RBF()) == 1
    assert G.slab_buffer_count(G.Matern52()) == 2
    assert G.slab_buffer_count(G.Sum(G.Scale(1.0, G.RBF()), G.Scale(1.0, G.Periodic()))) == 3
    assert G.is_stationary(G.RBF() * G.Periodic())
    assert not G.is_stationary(G.RBF() + G.Linear())


def test_lowering_preorder_and_rejects_custom_eval():
    k = G.parse_kernel("(+ (scale 2.0 (matern32 0.4)) (linear 0.5))")
    assert G.lower(k) == [("+", ()), ("scale", (2.0,)), ("matern32", (0.4,)), ("linear", (0.5,))]

    class CountingRBF(G.RBF):  # the reference's test_bench.py:118-123 pattern
        def _gram(self, x, y):
            return super()._gram(x, y)

    with pytest.raises(TypeError):
        G.lower(CountingRBF(0.5))

    class Plain(G.RBF):  # a subclass that keeps the evaluation lowers fine
        pass

    assert G.lower(Plain(0.5)) == [("rbf", (0.5,))]


def test_matvec_validation_before_device():
    x = np.ones((4, 1))
    with pytest.raises(G.DimensionMismatchError):
        G.matrix_free_matvec(G.RBF(1.0), x, 0.1, np.ones(5))
    with pytest.raises(ValueError):
        G.matrix_free_matvec(G.RBF(1.0), x, -0.1, np.ones(4))
    with pytest.raises(ValueError):
        G.matrix_free_matvec(G.RBF(1.0), x, 0.1, np.ones(4), block=0)
    with pytest.raises(G.NonFiniteError):
        G.matrix_free_matvec(G.RBF(1.0), x, 0.1, np.array([1.0, np.nan, 0, 0]))
    with pytest.raises(G.DimensionMismatchError):
        G.matrix_free_matvec(G.RBF(1.0), np.ones(4), 0.1, np.ones(4))


def test_fit_validation_and_scope():
    x = np.random.default_rng(0).random((10, 2))
    y = np.ones(10)
    with pytest.raises(ValueError):
        G.gp_fit(x, y, G.RBF(), 0.0, "cg")
    with pytest.raises(ValueError):
        G.gp_fit(x, y, G.RBF(), 0.1, "newton")
    with pytest.raises(G.DimensionMismatchError):
        G.gp_fit(x, y[:5], G.RBF(), 0.1, "cg")
    with pytest.raises(NotImplementedError):
        G.gp_fit(x, y, G.RBF(), 0.1, "cholesky")
    with pytest.raises(NotImplementedError):
        G.gp_fit(x, y, G.RBF(), 0.1, "auto")  # auto -> cholesky at N <= 4000


# ---- generic-callable CG / SLQ contract (reference test_solvers.py:104-216)

def test_cg_identity_one_iteration():
    b = np.random.default_rng(5).standard_normal(12)
    x, iters, res = G.cg_solve(lambda v: v, b)
    np.testing.assert_allclose(x, b, atol=1e-12)
    assert iters == 1 and res <= 1e-12 * np.linalg.norm(b)


def test_cg_zero_rhs_and_breakdown():
    x, iters, res = G.cg_solve(lambda v: v, np.zeros(6))
    assert iters == 0 and res == 0.0 and not x.any()
    with pytest.raises(G.OperatorNotSpdError):
        G.cg_solve(lambda v: -v, np.ones(4))


def test_cg_non_convergence_reported():
    rng = np.random.default_rng(7)
    a = rng.standard_normal((30, 30))
    a = a @ a.T + 0.01 * np.eye(30)
    x, iters, res = G.cg_solve(lambda v: a @ v, rng.standard_normal(30), G.CgConfig(max_iterations=2))
    assert iters == 2 and res > 0


def test_cg_config_validation():
    for kw in ({"rel_tolerance": 0.0}, {"probes": 0}, {"lanczos_steps": 0}, {"max_iterations": 0}):
        with pytest.raises(ValueError):
            G.CgConfig(**kw)


def test_slq_identity_diag_and_determinism():
    assert abs(G.slq_logdet(lambda v: v, 32, G.CgConfig(probes=8, lanczos_steps=10))) <= 1e-10
    d = np.random.default_rng(8).uniform(0.5, 4.0, 64)
    est = G.slq_logdet(lambda v: d * v, 64, G.CgConfig(probes=32, lanczos_steps=50))
    assert abs(est - np.log(d).sum()) / abs(np.log(d).sum()) <= 0.01
    d2 = np.linspace(1.0, 2.0, 16)
    a = G.slq_logdet(lambda v: d2 * v, 16, G.CgConfig(probes=4, lanczos_steps=8), seed=42)
    b = G.slq_logdet(lambda v: d2 * v, 16, G.CgConfig(probes=4, lanczos_steps=8), seed=42)
    assert a == b
    with pytest.raises(G.OperatorNotSpdError):
        G.slq_logdet(lambda v: -v, 16, G.CgConfig(probes=2, lanczos_steps=8))


def test_probe_block_matches_reference_recipe_and_prefix_stable():
    from oracle import gp_oracle as O

    z16 = G.probe_block(100, 16, 3)
    np.testing.assert_array_equal(z16, O.probes(100, 16, 3))
    np.testing.assert_array_equal(G.probe_block(100, 8, 3), z16[:, :8])
    assert set(np.unique(z16)) == {-1.0, 1.0}


def test_threaded_finite_scan_matches_numpy():
    """linalg's input check uses the library's threaded scan for large arrays
    (no GPU needed); it must agree with np.isfinite on NaN / +-Inf / huge."""
    from paper_2605_17898_b200 import _lib
    a = np.random.default_rng(0).standard_normal(3_000_001)
    assert _lib.all_finite(a)
    for pos in (0, 1_499_999, 3_000_000):
        for bad in (np.nan, np.inf, -np.inf):
            b = a.copy()
            b[pos] = bad
            assert not _lib.all_finite(b)
            with pytest.raises(G.NonFiniteError):
                G.linalg.as_vector(b)
    b = a.copy()
    b[7] = np.finfo(np.float64).max
    b[8] = -np.finfo(np.float64).tiny / 2  # subnormal
    assert _lib.all_finite(b)
    assert _lib.all_finite(np.empty(0))


def test_optimizer_matches_reference_bitwise():
    """optimize_hyperparams (models.py:362-413) is host logic: the reference's
    best point, centre trace and evaluation count on an analytic objective are
    reproduced exactly; flatten / unflatten_model_params likewise."""
    import math as _m

    g = golden("optimizer.npz")

    def toy(q):
        c = np.array([0.3, -1.2, 0.8])
        w = np.array([1.0, 0.5, 2.0])
        return float(-np.sum(w * (q - c) ** 2) + 0.1 * _m.sin(3.0 * q[0]) - 0.05 * q[1] * q[2])

    cfg = G.OptimizerConfig(steps=30, learning_rate=0.1)
    best, trace = G.optimize_hyperparams(toy, np.zeros(3), cfg)
    np.testing.assert_array_equal(best, g["toy_best"])
    np.testing.assert_array_equal(np.array(trace), g["toy_trace"])
    assert cfg.evaluations == int(g["toy_evals"]) == 30 * 7
    k = G.parse_kernel("(+ (scale 1.3 (rbf 0.6)) (matern52 0.9))")
    flat = G.flatten_model_params(k, 0.2)
    np.testing.assert_array_equal(flat, g["flat_values"])
    k2, noise2 = G.unflatten_model_params(k, flat + 0.1)
    assert G.format_kernel(k2) == str(g["flat_kernel2"]) and noise2 == float(g["flat_noise2"])
    with pytest.raises(G.DimensionMismatchError):
        G.unflatten_model_params(k, flat[:2])
    with pytest.raises(ValueError):
        G.OptimizerConfig(beta1=1.0)
    # a non-finite objective stops the run and returns the best point so far
    calls = []

    def bad(q):
        calls.append(1)
        return -float(np.sum(q * q)) if len(calls) < 5 else float("nan")

    best, trace = G.optimize_hyperparams(bad, np.ones(2), G.OptimizerConfig(steps=10))
    assert len(trace) == 1 and np.array_equal(best, np.ones(2))


def test_batched_optimizer_replays_exceptions_in_reference_order():
    """A batched objective evaluates all 2P + 1 points of a step at once; an
    evaluation that raises must surface only if the reference's sequential
    call order reaches it: here the first up-step is NaN, so
    the reference evaluates centre, up0, down0 and stops - the raising up1 is
    never reached."""

    class Obj:
        def __init__(self):
            self.seen = 0

        def __call__(self, q):
            raise AssertionError("the batch path must be used")

        def batch(self, qs, return_exceptions=False):
            self.seen += len(qs)
            out = []
            for i, q in enumerate(qs):
                if i == 1:
                    out.append(float("nan"))  # up0
                elif i == 3:
                    exc = ValueError("evaluation 3 fails")  # up1: never reached
                    if not return_exceptions:
                        raise exc
                    out.append(exc)
                else:
                    out.append(-float(np.sum(q * q)))
            return out

    cfg = G.OptimizerConfig(steps=4, learning_rate=0.1)
    obj = Obj()
    best, trace = G.optimize_hyperparams(obj, np.array([0.2, -0.1]), cfg)
    assert cfg.evaluations == 3 and len(trace) == 1 and obj.seen == 5
    np.testing.assert_array_equal(best, [0.2, -0.1])

    class Obj2(Obj):
        def batch(self, qs, return_exceptions=False):
            # the failing evaluation IS reached (it is the first up-step)
            return [-1.0] + [ValueError("reached")] * (len(qs) - 1)

    with pytest.raises(ValueError, match="reached"):
        G.optimize_hyperparams(Obj2(), np.array([0.2, -0.1]), G.OptimizerConfig(steps=2))
