"""Matrix-free K_y.V, CG and SLQ on the GPU (the hot path of minigp/solvers.py).

Public names and argument conventions follow the reference:

* ``matrix_free_matvec(kernel, x, noise, v, block=256)`` -> (K + noise I) v
  (solvers.py:57-84). ``v`` may also be an n x t block (multi-RHS extension);
  ``block`` keeps its validation but the device never holds a slab.
* ``cg_solve(apply, b, config)`` (solvers.py:87-123) and
  ``slq_logdet(apply, n, config, seed)`` (solvers.py:164-179) accept any
  callable ``apply``, exactly like the reference. When ``apply`` is a
  :class:`KernelOperator` — the operator ``gp_fit`` builds — the whole
  iteration runs on the device (``lgp_cg`` / ``lgp_lanczos``: every SLQ probe
  in lockstep through one multi-RHS matvec per step). A plain Python callable
  has no device representation, so its (O(n)-per-iteration) vector recurrence
  runs in NumPy around the caller's own ``apply``; that is the generic
  operator contract, not a fallback of the kernel hot path.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import scipy.linalg

from . import _lib
from .errors import DimensionMismatchError, OperatorNotSpdError
from .kernels import program, slab_buffer_count
from .linalg import _finite, as_block, as_matrix, as_vector, tracked


@dataclass
class CgConfig:
    """CG / SLQ settings (solvers.py:29-48); max_iterations None -> min(N, 1000)."""

    rel_tolerance: float = 1e-6
    max_iterations: int | None = None
    probes: int = 16
    lanczos_steps: int = 50

    def __post_init__(self):
        if not self.rel_tolerance > 0:
            raise ValueError("rel_tolerance must be positive")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.probes < 1 or self.lanczos_steps < 1:
            raise ValueError("probes and lanczos_steps must be at least 1")


class CgResult(NamedTuple):
    x: np.ndarray
    iterations: int
    final_residual: float


class KernelOperator:
    """The operator v -> (K(X, X) + noise I) v, resident on the GPU.

    Callable like the reference's ``apply`` closures (models.py:183,
    :208-210) — it returns a fresh NumPy array — but ``cg_solve`` and
    ``slq_logdet`` recognise it and keep their whole loop on the device.
    Points and the compiled kernel tree are uploaded once per operator.
    """

    def __init__(self, kernel, x, noise, ctx=None, _validated=False):
        self.kernel = kernel
        self.x = x if _validated else as_matrix(x, "X")
        self.noise = float(noise)
        self.n = self.x.shape[0]
        self.ctx = ctx if ctx is not None else _lib.default_context()
        self.prog = program(kernel)
        self.points = _lib.DevicePoints(self.ctx, self.x)

    def matvec(self, v):
        v = as_block(v, "v")
        if v.shape[0] != self.n:
            raise DimensionMismatchError(f"v has length {v.shape[0]}, X has {self.n} rows")
        return self._matvec(v)

    def _matvec(self, v, finite=True):
        # v: float64, C-contiguous, n rows; finite=False: the library checks v
        # on the host during its copy to the device (NonFiniteError)
        t = 1 if v.ndim == 1 else v.shape[1]
        out = _lib.result_buffer(v.shape)
        if self.n and t:
            _lib.check(_lib.lib().lgp_matvec(self.ctx.handle, self.prog.handle, self.points.handle,
                                             self.points.handle, self.noise, _lib.vptr(v), t,
                                             _lib.vptr(out), _lib.INPUTS_FINITE if finite else 0))
        return tracked(out)

    __call__ = matvec

    def cg(self, b, rel_tol, max_iter):
        b = as_block(b, "b")
        t = 1 if b.ndim == 1 else b.shape[1]
        x = np.empty(b.shape)
        iters = np.zeros(t, dtype=np.int32)
        res = np.zeros(t)
        mi = 0 if max_iter is None else int(max_iter)
        _lib.check(_lib.lib().lgp_cg(self.ctx.handle, self.prog.handle, self.points.handle,
                                     self.noise, _lib.vptr(b), t, float(rel_tol), mi,
                                     _lib.vptr(x), _lib.iptr(iters), _lib.dptr(res),
                                     _lib.INPUTS_FINITE))
        return x, iters, res

    def cg_shifted(self, b, shifts, rel_tol, max_iter):
        """Solutions of (K + (noise + shifts[e]) I) x_e = b for every shift
        (>= 0) with one matvec per iteration (lgp_cg_shifted, CG-M):
        (X [n x n_shifts], iterations, final residuals), each shift with the
        reference CG's stop rule of its own system."""
        b = as_block(b, "b")
        shifts = np.ascontiguousarray(shifts, dtype=np.float64)
        ns = shifts.shape[0]
        x = np.empty((b.shape[0], ns))
        iters = np.zeros(ns, dtype=np.int32)
        res = np.zeros(ns)
        mi = 0 if max_iter is None else int(max_iter)
        _lib.check(_lib.lib().lgp_cg_shifted(self.ctx.handle, self.prog.handle, self.points.handle,
                                             self.noise, _lib.vptr(b), ns, _lib.dptr(shifts),
                                             float(rel_tol), mi, _lib.vptr(x), _lib.iptr(iters),
                                             _lib.dptr(res), _lib.INPUTS_FINITE))
        return x, iters, res

    def lanczos(self, z, steps):
        z = np.ascontiguousarray(z, dtype=np.float64)
        t = z.shape[1]
        alphas = np.zeros((t, steps))
        betas = np.zeros((t, max(steps - 1, 1)))
        counts = np.zeros(t, dtype=np.int32)
        _lib.check(_lib.lib().lgp_lanczos(self.ctx.handle, self.prog.handle, self.points.handle,
                                          self.noise, _lib.vptr(z), t, int(steps),
                                          _lib.dptr(alphas), _lib.dptr(betas),
                                          _lib.iptr(counts), _lib.INPUTS_FINITE))
        return alphas, betas, counts


def matrix_free_matvec(kernel, x, noise, v, block=256):
    """(K + noise*I) @ v without materialising K (solvers.py:57-84).

    Kernel entries are generated on the GPU and reduced against ``v`` in
    registers; device memory stays O(N * t). ``v`` is an N-vector or an
    N x t block of right-hand sides.
    """
    # Finiteness: the reference checks X, then v, before anything else
    # (linalg.py:91-106). On the success path of a large call the scans move
    # into the library, off the critical path: X is checked on the device
    # during its upload (point statistics), v on the host while its
    # host->device copy is in flight. Every error branch below runs the host
    # scans first, so the reference's error order is kept.
    x = as_matrix(x, "X", check=False)
    v = as_block(v, "v", check=False)
    defer = x.size + v.size >= (1 << 18)

    def scans():
        _finite(x, "X")
        _finite(v, "v")

    if not defer:
        scans()
    n = x.shape[0]
    if v.shape[0] != n:
        scans()
        raise DimensionMismatchError(f"v has length {v.shape[0]}, X has {n} rows")
    noise = float(noise)
    if not np.isfinite(noise) or noise < 0:
        scans()
        raise ValueError("noise must be finite and nonnegative")
    if block < 1:
        scans()
        raise ValueError("block must be at least 1")
    try:
        slab_buffer_count(kernel)  # node-protocol check, as the reference does per call
        op = KernelOperator(kernel, x, noise, _validated=True)
    except Exception:
        if defer:
            scans()  # NonFiniteError takes precedence, as in the reference
        raise
    return op._matvec(v, finite=not defer)


def cg_solve(apply, b, config=None):
    """Unpreconditioned CG for SPD operators (solvers.py:87-123).

    Stops when sqrt(r.r) <= rel_tolerance * ||b|| or at max_iterations
    (reported, not raised); pAp <= 0 raises OperatorNotSpdError.
    """
    cfg = config if config is not None else CgConfig()
    b = as_vector(b, "b")
    if isinstance(apply, KernelOperator):
        if b.shape[0] != apply.n:
            raise DimensionMismatchError(f"b has length {b.shape[0]}, operator order {apply.n}")
        x, iters, res = apply.cg(b, cfg.rel_tolerance, cfg.max_iterations)
        return CgResult(tracked(x), int(iters[0]), float(res[0]))
    return _cg_callable(apply, b, cfg)


def _cg_callable(apply, b, cfg):
    # generic-callable contract: the caller's own apply(), reference recurrence
    n = b.shape[0]
    max_iter = cfg.max_iterations if cfg.max_iterations is not None else min(n, 1000)
    x = tracked(np.zeros(n))
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return CgResult(x, 0, 0.0)
    tol = cfg.rel_tolerance * bnorm
    r = tracked(b.copy())
    p = tracked(b.copy())
    rs = float(r @ r)
    k = 0
    for k in range(1, max_iter + 1):
        ap = apply(p)
        pap = float(p @ ap)
        if pap <= 0.0:
            raise OperatorNotSpdError(f"CG breakdown: p.A.p = {pap:g} is not positive")
        step = rs / pap
        x += step * p
        r -= step * ap
        rs_new = float(r @ r)
        if np.sqrt(rs_new) <= tol:
            return CgResult(x, k, float(np.sqrt(rs_new)))
        p *= rs_new / rs
        p += r
        rs = rs_new
    return CgResult(x, k, float(np.sqrt(rs)))


def probe_block(n, count, seed):
    """Rademacher probes exactly as slq_logdet draws them (solvers.py:175-177):
    one PCG64 child stream per probe, so the first k of `count` probes do not
    depend on `count`."""
    z = np.empty((n, count))
    kids = np.random.SeedSequence(seed).spawn(count)

    def draw(c):
        rng = np.random.Generator(np.random.PCG64(kids[c]))
        z[:, c] = rng.integers(0, 2, size=n) * 2.0 - 1.0

    if n * count < (1 << 18) or count == 1:
        for c in range(count):
            draw(c)
    else:  # independent streams; the ufunc / strided column writes release the GIL
        list(_probe_pool().map(draw, range(count)))
    return z


_POOL = None


def _probe_pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1)))
    return _POOL


def gauss_quadrature(alphas, betas):
    """sum_i tau_1i^2 log(lambda_i) of the Lanczos tridiagonal (solvers.py:155-161)."""
    lam, vec = scipy.linalg.eigh_tridiagonal(alphas, betas)
    if lam.min() <= 0.0:
        raise OperatorNotSpdError(
            f"nonpositive Ritz value {lam.min():g}; operator is not positive definite")
    tau = vec[0]
    return float(np.sum(tau * tau * np.log(lam)))


def slq_logdet(apply, n, config=None, seed=0):
    """Stochastic Lanczos quadrature estimate of log det(A) (solvers.py:164-179).

    For a KernelOperator all probes advance in lockstep on the device: each
    Lanczos step is ONE multi-RHS matvec (t = probes) instead of `probes`
    separate ones; the tiny eigenproblems stay on the host as in the
    reference.
    """
    cfg = config if config is not None else CgConfig()
    steps = min(cfg.lanczos_steps, n)
    z = probe_block(n, cfg.probes, seed)
    if isinstance(apply, KernelOperator):
        if apply.n != n:
            raise DimensionMismatchError(f"operator order {apply.n} != n={n}")
        total = 0.0
        for c0 in range(0, cfg.probes, 256):
            zc = z[:, c0:c0 + 256]
            al, be, cnt = apply.lanczos(zc, steps)
            for c in range(zc.shape[1]):
                m = int(cnt[c])
                total += n * gauss_quadrature(al[c, :m], be[c, :m - 1])
        return total / cfg.probes
    total = 0.0
    for c in range(cfg.probes):
        total += n * _lanczos_callable(apply, np.ascontiguousarray(z[:, c]), steps)
    return total / cfg.probes


class _ShiftFallback(Exception):
    """A shifted member's Lanczos would run past the seed's early exit."""


def slq_logdet_shifted(op, n, config, seed, members):
    """slq_logdet of c_e (A + sig_e I) for every member (c_e, sig_e), A = op,
    from ONE device Lanczos run on A: Lanczos is shift- and scale-invariant
    (same basis; alpha -> c (alpha + sig), beta -> c beta), so each member's
    tridiagonal - including the reference's early exit (solvers.py:151-152),
    re-evaluated on the member's own coefficients - and its quadrature
    (solvers.py:155-161) follow from the seed's. Returns one log-det or
    OperatorNotSpdError per member; raises _ShiftFallback if a member would
    continue past a probe's early exit on A."""
    cfg = config if config is not None else CgConfig()
    steps = min(cfg.lanczos_steps, n)
    z = probe_block(n, cfg.probes, seed)
    al, be, cnt = [], [], []
    for c0 in range(0, cfg.probes, 256):
        a, b, m = op.lanczos(z[:, c0:c0 + 256], steps)
        al.append(a)
        be.append(b)
        cnt.append(m)
    al, be, cnt = np.vstack(al), np.vstack(be), np.concatenate(cnt)
    out = []
    for c, sig in members:
        total = 0.0
        try:
            for p in range(cfg.probes):
                m = int(cnt[p])
                a = c * (al[p, :m] + sig)
                b = c * be[p, :max(m - 1, 0)]
                cut = m
                for j in range(m - 1):
                    if b[j] <= 1e-12 * max(1.0, abs(a[j])):
                        cut = j + 1
                        break
                if cut == m and m < steps:
                    raise _ShiftFallback()
                total += n * gauss_quadrature(a[:cut], b[:cut - 1])
            out.append(total / cfg.probes)
        except OperatorNotSpdError as exc:
            out.append(exc)
    return out


def _lanczos_callable(apply, z, steps):
    # generic-callable contract (solvers.py:126-161)
    q = z / np.linalg.norm(z)
    basis = tracked(np.zeros((steps, z.shape[0])))
    al, be = [], []
    for j in range(steps):
        basis[j] = q
        w = apply(q)
        a = float(q @ w)
        al.append(a)
        w = w - a * q
        if j > 0:
            w -= be[-1] * basis[j - 1]
        act = basis[: j + 1]
        w -= act.T @ (act @ w)
        if j == steps - 1:
            break
        nb = float(np.linalg.norm(w))
        if nb <= 1e-12 * max(1.0, abs(a)):
            break
        be.append(nb)
        q = w / nb
    return gauss_quadrature(np.array(al), np.array(be))
