"""Exact GP regression through the matrix-free CG path (minigp/models.py, CG branch).

``gp_fit(..., strategy="cg")``, ``gp_predict`` and ``log_marginal_likelihood``
keep the reference's signatures, validation and fitted-state fields
(models.py:52-72, 143-266). The operator is always the GPU-resident
:class:`KernelOperator` (the reference switches to a dense Gram below
N = 2048, models.py:174-182; the two operators are the same matrix, only
rounding differs), so:

* fit        -> one device CG solve (lgp_cg)
* predict    -> mean from the fused cross matvec K(X*, X) alpha; variance from
                k* formed on the device and ONE multi-RHS device CG with one
                column per test point (the reference runs T separate solves,
                models.py:239-246)
* evidence   -> y.alpha + SLQ log-det with all probes in lockstep (lgp_lanczos)

The Cholesky, SKI and sparse-variational strategies are outside this
drop-in's scope and raise NotImplementedError.
"""

from __future__ import annotations

import math
import warnings
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DimensionMismatchError
from .kernels import is_stationary
from .linalg import as_matrix, as_vector, tracked
from .solvers import CgConfig, KernelOperator, cg_solve

AUTO_CHOLESKY_MAX = 4000  # models.py:43
DENSE_OPERATOR_MAX = 2048  # models.py:44 (kept for reference; the device never densifies)
CG_FIT_BLOCK = 32  # models.py:45
FIT_CG_TOLERANCE = 1e-8  # models.py:46
LOG_2PI = math.log(2.0 * math.pi)


@dataclass(frozen=True)
class ExactState:
    """Fitted exact GP (models.py:52-72); ``operator`` holds the device operator."""

    x_train: np.ndarray
    y_train: np.ndarray
    kernel: object
    noise: float
    strategy: str
    alpha: np.ndarray
    factor: object = None
    gram_y: np.ndarray | None = None
    ski: object = None
    cg_iterations: int | None = None
    cg_final_residual: float | None = None
    cg_config: CgConfig | None = None
    operator: KernelOperator | None = field(default=None, repr=False, compare=False)


def _check_noise(noise):
    noise = float(noise)
    if not math.isfinite(noise) or noise <= 0:
        raise ValueError("noise variance must be positive and finite")
    return noise


def _resolve_strategy(strategy, n, d, kernel):
    s = str(strategy).lower()
    if s == "auto":  # models.py:130-140
        if n <= AUTO_CHOLESKY_MAX:
            s = "cholesky"
        elif d == 1 and is_stationary(kernel):
            s = "ski"
        else:
            s = "cg"
    if s not in ("cholesky", "cg", "ski"):
        raise ValueError(f"unknown strategy {strategy!r}")
    if s != "cg":
        raise NotImplementedError(
            f"strategy {s!r} is outside this drop-in's scope: only the matrix-free CG path "
            "is provided (pass strategy='cg')")
    return s


def gp_fit(x, y, kernel, noise, strategy="auto", *, cg_config=None, grid_size=None, ctx=None):
    """Fit an exact GP with the device CG solver (models.py:143-200). ``ctx``:
    the library context (GPU / stream) to run on, default the process's.

    Only the matrix-free CG path is provided: ``strategy`` must be ``"cg"``,
    or ``"auto"`` where the reference resolves it to CG (N > 4000 and not a
    1-D stationary kernel, models.py:130-140). The reference's Cholesky and
    SKI strategies (the default ``"auto"`` for N <= 4000) raise
    ``NotImplementedError`` rather than fall back to a CPU path. Unlike the
    reference, N <= 2048 also uses the matrix-free operator (the reference
    switches to a dense Gram there, models.py:174-182)."""
    x = as_matrix(x, "X")
    y = as_vector(y, "y")
    n, d = x.shape
    if y.shape[0] != n:
        raise DimensionMismatchError(f"y has length {y.shape[0]}, X has {n} rows")
    if n < 1:
        raise DimensionMismatchError("need at least one training point")
    noise = _check_noise(noise)
    resolved = _resolve_strategy(strategy, n, d, kernel)
    cfg = cg_config if cg_config is not None else CgConfig(rel_tolerance=FIT_CG_TOLERANCE)
    op = KernelOperator(kernel, x, noise, ctx=ctx)
    res = cg_solve(op, y, cfg)
    return ExactState(x, y, kernel, noise, resolved, res.x, cg_iterations=res.iterations,
                      cg_final_residual=res.final_residual, cg_config=cfg, operator=op)


def _operator(state):
    """The fitted K_y operator (models.py:203-213)."""
    if state.operator is not None:
        return state.operator
    return KernelOperator(state.kernel, state.x_train, state.noise)


def gp_predict(state, x_star):
    """Posterior mean and latent variance (models.py:216-250)."""
    x_star = as_matrix(x_star, "X*")
    if x_star.shape[1] != state.x_train.shape[1]:
        raise DimensionMismatchError(
            f"test inputs have {x_star.shape[1]} columns, training had {state.x_train.shape[1]}")
    t = x_star.shape[0]
    if t == 0:
        return tracked(np.zeros(0)), tracked(np.zeros(0))
    op = _operator(state)
    lib, ctx = _lib.lib(), op.ctx
    test = _lib.DevicePoints(ctx, x_star)
    alpha = np.ascontiguousarray(state.alpha)
    mean = np.empty(t)
    _lib.check(lib.lgp_matvec(ctx.handle, op.prog.handle, test.handle, op.points.handle, 0.0,
                              _lib.vptr(alpha), 1, _lib.vptr(mean), 0))
    prior = np.empty(t)
    _lib.check(lib.lgp_diag(ctx.handle, op.prog.handle, test.handle, _lib.vptr(prior), 0))
    cfg = state.cg_config if state.cg_config is not None else CgConfig()
    quad = np.empty(t)
    iters = np.zeros(t, dtype=np.int32)
    res = np.zeros(t)
    mi = 0 if cfg.max_iterations is None else int(cfg.max_iterations)
    _lib.check(lib.lgp_predict_quad(ctx.handle, op.prog.handle, op.points.handle, test.handle,
                                    state.noise, cfg.rel_tolerance, mi, _lib.dptr(quad),
                                    _lib.iptr(iters), _lib.dptr(res)))
    cap = mi if mi > 0 else min(state.x_train.shape[0], 1000)
    capped = int(np.count_nonzero(iters >= cap))
    if capped:
        # the reference reports a non-converged solve instead of raising
        # (solvers.py:122-123) and gp_predict ignores it; say so
        warnings.warn(f"gp_predict: the variance CG of {capped} of {t} test points stopped at the "
                      f"{cap}-iteration budget (tolerance {cfg.rel_tolerance:g} not reached)",
                      RuntimeWarning, stacklevel=2)
    var = prior - quad
    np.maximum(var, 0.0, out=var)
    return tracked(mean), tracked(var)


def log_marginal_likelihood(state, seed=0):
    """-1/2 (y.alpha + log det K_y + N log 2 pi), log-det by device SLQ (models.py:253-266)."""
    from .solvers import slq_logdet

    n = state.y_train.shape[0]
    quad = float(state.y_train @ state.alpha)
    cfg = state.cg_config if state.cg_config is not None else CgConfig()
    ld = slq_logdet(_operator(state), n, cfg, seed=seed)
    return -0.5 * (quad + ld + n * LOG_2PI)


# ------------------------------------------- hyper-parameter optimisation
# (the caller of the fit + evidence path). Host-side
# restatement of minigp/models.py:89-111 and :347-413; every objective
# evaluation runs the device fit (lgp_cg) and SLQ evidence (lgp_lanczos).

@dataclass
class OptimizerConfig:
    """Adam on central finite differences (models.py:89-111). `evaluations`
    is written by optimize_hyperparams: steps * (2P + 1) calls."""

    steps: int = 100
    learning_rate: float = 0.05
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    fd_epsilon: float = 1e-4
    evaluations: int = 0

    def __post_init__(self):
        if self.steps < 0:
            raise ValueError("steps must be nonnegative")
        if min(self.learning_rate, self.fd_epsilon, self.eps) <= 0:
            raise ValueError("learning_rate, fd_epsilon and eps must be positive")
        if not (0 < self.beta1 < 1 and 0 < self.beta2 < 1):
            raise ValueError("beta coefficients must lie in (0, 1)")


def flatten_model_params(kernel, noise):
    """Log-space vector [kernel hyperparameters..., log noise] (models.py:347-349)."""
    from .kernels import flatten_params

    return tracked(np.append(flatten_params(kernel), math.log(noise)))


def unflatten_model_params(kernel, values):
    """(kernel, noise) from a flatten_model_params vector (models.py:352-359)."""
    from .kernels import n_params, unflatten_params

    values = np.asarray(values, dtype=np.float64)
    want = n_params(kernel) + 1
    if values.shape != (want,):
        raise DimensionMismatchError(f"expected {want} values, got {values.shape}")
    return unflatten_params(kernel, values[:-1]), float(np.exp(values[-1]))


def optimize_hyperparams(objective, p0, config):
    """Maximise `objective` over a log-space vector (models.py:362-413).

    Adam ascent on a central-difference gradient: per step one centre call and
    two per coordinate (2P + 1). A non-finite value stops the run; returns the
    best centre seen and the trace of centre values.
    """
    p = np.array(p0, dtype=np.float64, copy=True)
    if p.ndim != 1:
        raise DimensionMismatchError("parameter vector must be 1-d")
    config.evaluations = 0

    def call(q):
        config.evaluations += 1
        return float(objective(q))

    dim = p.shape[0]
    m1 = np.zeros(dim)
    m2 = np.zeros(dim)
    trace, best_p, best = [], p.copy(), -np.inf
    h = config.fd_epsilon
    batch = getattr(objective, "batch", None)
    for step in range(1, config.steps + 1):
        if batch is not None:
            # the 2P + 1 evaluations of this step at once (concurrently on the
            # device); the sequential call order below replays on the values,
            # so the result and the evaluation count are the reference's
            pts = [p.copy()]
            for i in range(dim):
                for sgn in (1.0, -1.0):
                    q = p.copy()
                    q[i] = p[i] + sgn * h
                    pts.append(q)
            # each point's value, or the exception its evaluation raised: an
            # exception surfaces only when the replayed sequential order
            # reaches that point (the reference stops at the first non-finite
            # value and never evaluates the rest)
            vals = iter(batch(pts, return_exceptions=True))

            def call(q, _vals=vals):
                config.evaluations += 1
                v = next(_vals)
                if isinstance(v, BaseException):
                    raise v
                return float(v)
        centre = call(p)
        if not math.isfinite(centre):
            break
        trace.append(centre)
        if centre > best:
            best, best_p = centre, p.copy()
        grad = np.empty(dim)
        ok = True
        for i in range(dim):
            q = p.copy()
            q[i] += h
            up = call(q)
            q[i] = p[i] - h
            down = call(q)
            if not (math.isfinite(up) and math.isfinite(down)):
                ok = False
                break
            grad[i] = (up - down) / (2.0 * h)
        if not ok:
            break
        m1 = config.beta1 * m1 + (1.0 - config.beta1) * grad
        m2 = config.beta2 * m2 + (1.0 - config.beta2) * grad * grad
        m1_hat = m1 / (1.0 - config.beta1**step)
        m2_hat = m2 / (1.0 - config.beta2**step)
        p = p + config.learning_rate * m1_hat / (np.sqrt(m2_hat) + config.eps)
    return tracked(best_p), trace


def _peel_root_scale(kernel):
    """(c, inner): kernel = c * inner for the chain of Scale nodes at the root
    (c = 1 without one)."""
    from .kernels import Scale

    c = 1.0
    while isinstance(kernel, Scale):
        c *= float(kernel.outputscale)
        kernel = kernel.child
    return c, kernel


class _EvidenceObjective:
    """q -> log marginal likelihood of gp_fit(x, y, *unflatten_model_params(
    kernel, q), "cg"). ``batch(qs)`` evaluates several parameter vectors at
    once (an optimiser step's 2P + 1 points):

    * points whose kernels differ only in the root output scale c and whose
      noise differs (centre, +-scale, +-noise) share ONE operator family
      c (K1 + lam I), lam = noise / c: their fits are one multi-shift CG on K1
      (lgp_cg_shifted: one matvec per iteration for all of them) and their
      log-dets one device Lanczos run (shift / scale invariance,
      solvers.slq_logdet_shifted) - SURVEY.md §8f row 3;
    * the other points (e.g. +-lengthscale) are single evaluations;
    * groups / singletons run concurrently, one host thread and one library
      context (own CUDA stream) per worker.

    A fused value agrees with the separate evaluation to the CG's rounding
    (~1e-10 relative, tests/test_gpu_solvers.py); ``fuse_shifts=False`` gives
    bit-identical separate evaluations."""

    def __init__(self, x, y, kernel, cg_config, seed, workers, fuse_shifts=True):
        self.x, self.y, self.kernel = x, y, kernel
        self.cg_config, self.seed = cg_config, seed
        self.workers = workers
        self.fuse_shifts = fuse_shifts
        self._pool = None
        self._ctx = threading.local()

    def _eval(self, q, ctx=None):
        k, noise = unflatten_model_params(self.kernel, q)
        st = gp_fit(self.x, self.y, k, noise, "cg", cg_config=self.cg_config, ctx=ctx)
        return log_marginal_likelihood(st, seed=self.seed)

    def _eval_group(self, qs, ctx=None):
        """Log marginal likelihoods of points that share K1 (see the class
        doc); one value or exception per point."""
        from .solvers import _ShiftFallback, slq_logdet_shifted

        mem = []
        for q in qs:
            k, noise = unflatten_model_params(self.kernel, q)
            mem.append((_peel_root_scale(k), _check_noise(noise)))
        k1 = mem[0][0][1]
        c = np.array([m[0][0] for m in mem])
        lam = np.array([m[1] for m in mem]) / c
        s = int(np.argmin(lam))
        cfg = self.cg_config if self.cg_config is not None else CgConfig(rel_tolerance=FIT_CG_TOLERANCE)
        op = KernelOperator(k1, self.x, float(lam[s]), ctx=ctx, _validated=True)
        try:
            X, _, _ = op.cg_shifted(self.y, lam - lam[s], cfg.rel_tolerance, cfg.max_iterations)
            lds = slq_logdet_shifted(op, self.x.shape[0], cfg, self.seed,
                                     [(float(c[e]), float(lam[e] - lam[s])) for e in range(len(qs))])
        except _ShiftFallback:
            return [self._eval(q, ctx) for q in qs]
        n = self.x.shape[0]
        out = []
        for e in range(len(qs)):
            if isinstance(lds[e], BaseException):
                out.append(lds[e])
                continue
            alpha = X[:, e] / c[e]
            out.append(-0.5 * (float(self.y @ alpha) + lds[e] + n * LOG_2PI))
        return out

    def __call__(self, q):
        return self._eval(q)

    def _worker_ctx(self):
        ctx = getattr(self._ctx, "ctx", None)
        if ctx is None:
            ctx = self._ctx.ctx = _lib.Context(_lib.default_context().device)
        return ctx

    def batch(self, qs, return_exceptions=False):
        """Values of every q; with return_exceptions an evaluation that raises
        yields its exception in place of its value."""
        def guard(v):
            if isinstance(v, BaseException) and not return_exceptions:
                raise v
            return v

        # tasks: groups of points sharing K1 (fused) and single points
        tasks = []
        if self.fuse_shifts and len(qs) > 1:
            from .kernels import format_kernel

            groups = {}
            for i, q in enumerate(qs):
                k, _ = unflatten_model_params(self.kernel, q)
                groups.setdefault(format_kernel(_peel_root_scale(k)[1]), []).append(i)
            tasks = list(groups.values())
        else:
            tasks = [[i] for i in range(len(qs))]

        def run(idxs, ctx=None):
            try:
                if len(idxs) == 1:
                    return [self._eval(qs[idxs[0]], ctx)]
                return self._eval_group([qs[i] for i in idxs], ctx)
            except Exception as exc:  # noqa: BLE001 (returned, re-raised below)
                return [exc] * len(idxs)

        if self.workers <= 1 or len(tasks) <= 1:
            results = [run(idxs) for idxs in tasks]
        else:
            if self._pool is None:
                self._pool = ThreadPoolExecutor(max_workers=self.workers)
            results = list(self._pool.map(lambda idxs: run(idxs, self._worker_ctx()), tasks))
        out = [None] * len(qs)
        for idxs, vals in zip(tasks, results):
            for i, v in zip(idxs, vals):
                out[i] = v
        return [guard(v) for v in out]


def exact_evidence_objective(x, y, kernel, cg_config=None, seed=0, workers=None, fuse_shifts=True):
    """The exact-GP objective for optimize_hyperparams: each call one device CG
    fit and one device SLQ evidence (the kernel program is cached by tree
    shape, parameters are launch arguments). ``batch`` (what the optimiser
    uses) fuses the points that differ only in the root output scale and the
    noise into one multi-shift CG + one Lanczos run (``fuse_shifts``), and
    ``workers`` concurrent contexts evaluate the remaining tasks at once
    (default min(8, 2P+1) for N >= 8192, else 1; tools/optimizer_timing.py)."""
    x = as_matrix(x, "X")
    y = as_vector(y, "y")
    if workers is None:
        from .kernels import n_params

        # concurrency pays once the device work dominates: 3 Adam steps at
        # N = 20000 1.45 vs 2.76 s; at N <= 4000 host time dominates (equal)
        workers = min(8, 2 * (n_params(kernel) + 1) + 1) if x.shape[0] >= 8192 else 1
    return _EvidenceObjective(x, y, kernel, cg_config, seed, int(workers), fuse_shifts)


def metrics(mean, var_latent, noise, y_true):
    """(rmse, mean negative log predictive density, 95 % coverage) of latent
    predictions scored against noisy observations (models.py:471-487): the
    noise variance is added to the latent variance before scoring. Host-side
    caller of gp_predict's outputs (the JSON server's ``metrics`` op)."""
    mean = as_vector(mean, "mean")
    var_latent = as_vector(var_latent, "var")
    y_true = as_vector(y_true, "y")
    if not (mean.shape == var_latent.shape == y_true.shape):
        raise DimensionMismatchError("metrics inputs must share length")
    s2 = var_latent + float(noise)
    resid = y_true - mean
    sq = resid * resid
    rmse = float(np.sqrt(np.mean(sq)))
    nll = float(np.mean(0.5 * np.log(2.0 * math.pi * s2) + sq / (2.0 * s2)))
    cover = float(np.mean(np.abs(resid) <= 1.96 * np.sqrt(s2)))
    return rmse, nll, cover
