"""CPU oracle for the matrix-free K_y.V / CG / SLQ hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker. It restates, in float64 NumPy, the reference
algorithm of ``minigp`` (the Python package under ``/root/reference/pkg/src``)
for exactly the functions on the hot path, so that the CUDA product path can be
checked on the GPU box, where the reference itself is absent.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it. The product package
(``paper_2605_17898_b200``) never does; it fails loudly without its CUDA
library instead of falling back here.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (imported from
``/root/reference`` in the build container) and stores its outputs under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this oracle against
every fixture (bit-for-bit where the operation order is the same, else to
1e-12).  The oracle is therefore *pinned* to the reference.

Kernel trees are consumed in the same lowered form the device library
compiles: a pre-order list of ``(kind, params)`` nodes (see
``paper_2605_17898_b200.kernels.lower``), kind names ``rbf``, ``matern12``,
``matern32``, ``matern52``, ``periodic``, ``linear``, ``scale``, ``+``, ``*``.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

SQRT3 = math.sqrt(3.0)
SQRT5 = math.sqrt(5.0)
LOG_2PI = math.log(2.0 * math.pi)

ARITY = {"rbf": 0, "matern12": 0, "matern32": 0, "matern52": 0, "periodic": 0,
         "linear": 0, "scale": 1, "+": 2, "*": 2}


class OracleNotSpd(RuntimeError):
    """Mirror of minigp.errors.OperatorNotSpdError (errors.py:41-42)."""


# --------------------------------------------------------------------------- trees

def parse_tree(text):
    """s-expression -> pre-order node list.  Grammar of kernels.py:445-513."""
    toks = text.replace("(", " ( ").replace(")", " ) ").split()
    nodes = []
    pos = 0

    def walk():
        nonlocal pos
        assert toks[pos] == "("
        head = toks[pos + 1]
        pos += 2
        if head in ("rbf", "matern12", "matern32", "matern52", "linear"):
            nodes.append((head, (float(toks[pos]),)))
            pos += 1
        elif head == "periodic":
            nodes.append((head, (float(toks[pos]), float(toks[pos + 1]))))
            pos += 2
        elif head == "scale":
            nodes.append((head, (float(toks[pos]),)))
            pos += 1
            walk()
        elif head in ("+", "*"):
            nodes.append((head, ()))
            walk()
            walk()
        else:
            raise ValueError(head)
        assert toks[pos] == ")"
        pos += 1

    walk()
    return nodes


def _subtree_end(nodes, i):
    need = 1
    while need:
        need += ARITY[nodes[i][0]] - 1
        i += 1
    return i


def slab_buffers(nodes, i=0):
    """Peak live slab buffers; kernels.py:79-80,147-148,185-186,231-232,305,339-340."""
    kind = nodes[i][0]
    if kind in ("rbf", "matern12", "linear"):
        return 1
    if kind in ("matern32", "matern52", "periodic"):
        return 2
    if kind == "scale":
        return slab_buffers(nodes, i + 1)
    j = _subtree_end(nodes, i + 1)
    return max(slab_buffers(nodes, i + 1), 1 + slab_buffers(nodes, j))


# --------------------------------------------------------------- dense primitives

def sqdist(x, y, same=False):
    """Distance trick of linalg.py:207-235 (norms + one product, clamp, symmetrise)."""
    xn = np.einsum("ij,ij->i", x, x)
    yn = xn if same else np.einsum("ij,ij->i", y, y)
    out = x @ np.ascontiguousarray(y.T)  # linalg.py:121-127 copies the transpose
    out *= -2.0
    out += xn[:, None]
    out += yn[None, :]
    np.maximum(out, 0.0, out=out)
    if same:
        sym = out + out.T
        sym *= 0.5
        np.fill_diagonal(sym, 0.0)
        out = sym
    return out


def gram(nodes, x, y, same=False, i=0):
    """k(x_a, y_b) for the subtree rooted at nodes[i].

    Leaf closed forms follow kernels.py: RBF :65-68, Matern12 :95-99,
    Matern32 :126-136, Matern52 :163-174, Periodic :203-220, Linear :247-256;
    combinators Scale :288-291, Sum :322-326, Product :357-361.
    """
    kind, prm = nodes[i]
    if kind == "rbf":
        g = sqdist(x, y, same)
        g *= -0.5 / prm[0] ** 2
        return np.exp(g, out=g)
    if kind == "matern12":
        g = sqdist(x, y, same)
        np.sqrt(g, out=g)
        g *= -1.0 / prm[0]
        return np.exp(g, out=g)
    if kind == "matern32":
        g = sqdist(x, y, same)
        np.sqrt(g, out=g)
        g *= SQRT3 / prm[0]
        e = np.exp(-g)
        g += 1.0
        g *= e
        return g
    if kind == "matern52":
        g = sqdist(x, y, same)
        g *= 5.0 / prm[0] ** 2
        r = np.sqrt(g)
        g /= 3.0
        g += r
        g += 1.0
        g *= np.exp(-r)
        return g
    if kind == "periodic":
        ell, per = prm
        acc = np.zeros((x.shape[0], y.shape[0]))
        for d in range(x.shape[1]):
            w = np.subtract(x[:, d, None], y[None, :, d])
            w *= math.pi / per
            np.sin(w, out=w)
            np.square(w, out=w)
            acc += w
        if same:
            sym = acc + acc.T
            sym *= 0.5
            np.fill_diagonal(sym, 0.0)
            acc = sym
        acc *= -2.0 / ell ** 2
        return np.exp(acc, out=acc)
    if kind == "linear":
        g = x @ np.ascontiguousarray(y.T)
        g *= prm[0]
        if same:
            s = g + g.T
            s *= 0.5
            return s
        return g
    if kind == "scale":
        g = gram(nodes, x, y, same, i + 1)
        g *= prm[0]
        return g
    j = _subtree_end(nodes, i + 1)
    a = gram(nodes, x, y, same, i + 1)
    b = gram(nodes, x, y, same, j)
    if kind == "+":
        a += b
    else:
        a *= b
    return a


def diag(nodes, x, i=0):
    """kernel_diag (kernels.py:398-400) via the per-node _diag rules."""
    kind, prm = nodes[i]
    if kind in ("rbf", "matern12", "matern32", "matern52", "periodic"):
        return np.ones(x.shape[0])
    if kind == "linear":
        d = np.einsum("ij,ij->i", x, x)
        d *= prm[0]
        return d
    if kind == "scale":
        d = diag(nodes, x, i + 1)
        d *= prm[0]
        return d
    j = _subtree_end(nodes, i + 1)
    a = diag(nodes, x, i + 1)
    if kind == "+":
        a += diag(nodes, x, j)
    else:
        a *= diag(nodes, x, j)
    return a


# ------------------------------------------------------------------ hot path

def matvec(nodes, x, noise, v, block=256, row_range=None):
    """(K + noise I) v by row slabs, solvers.py:57-84.

    ``v`` may be N x t; each column is then done separately, exactly as t
    calls of the single-vector reference would (the reference has no
    multi-RHS path).  ``row_range=(r0, r1)`` returns only those output rows
    (the loop body is row-separable, solvers.py:77-81); used for full-size
    parity on row subsets.
    """
    x = np.ascontiguousarray(x, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    cols = v[:, None] if v.ndim == 1 else v
    n = x.shape[0]
    r0, r1 = (0, n) if row_range is None else row_range
    rows = max(1, int(block) // slab_buffers(nodes))
    out = np.empty((r1 - r0, cols.shape[1]))
    for c in range(cols.shape[1]):
        vc = np.ascontiguousarray(cols[:, c])
        oc = np.empty(r1 - r0)
        for a in range(r0, r1, rows):
            b = min(a + rows, r1)
            slab = gram(nodes, x[a:b], x)
            np.dot(slab, vc, out=oc[a - r0:b - r0])
        if noise != 0.0:
            oc += noise * vc[r0:r1]
        out[:, c] = oc
    return out[:, 0] if v.ndim == 1 else out


def cg(apply, b, rel_tol=1e-6, max_iter=None):
    """Unpreconditioned CG with the recurrence-residual stop, solvers.py:87-123.

    Returns (x, iterations, final_residual)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = b.shape[0]
    max_iter = max_iter if max_iter is not None else min(n, 1000)
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, 0.0
    tol = rel_tol * bnorm
    r = b.copy()
    p = b.copy()
    rs = float(r @ r)
    it = 0
    for it in range(1, max_iter + 1):
        ap = apply(p)
        pap = float(p @ ap)
        if pap <= 0.0:
            raise OracleNotSpd(f"p.A.p = {pap:g}")
        step = rs / pap
        x += step * p
        r -= step * ap
        rs_new = float(r @ r)
        if np.sqrt(rs_new) <= tol:
            return x, it, float(np.sqrt(rs_new))
        p *= rs_new / rs
        p += r
        rs = rs_new
    return x, it, float(np.sqrt(rs))


def lanczos(apply, z, steps):
    """Lanczos with one CGS re-orthogonalisation pass per step, solvers.py:126-154.

    Returns (alphas, betas) of the tridiagonal actually built."""
    q = z / np.linalg.norm(z)
    basis = np.zeros((steps, z.shape[0]))
    alphas, betas = [], []
    for j in range(steps):
        basis[j] = q
        w = apply(q)
        a = float(q @ w)
        alphas.append(a)
        w = w - a * q
        if j > 0:
            w -= betas[-1] * basis[j - 1]
        act = basis[: j + 1]
        w -= act.T @ (act @ w)
        if j == steps - 1:
            break
        nb = float(np.linalg.norm(w))
        if nb <= 1e-12 * max(1.0, abs(a)):
            break
        betas.append(nb)
        q = w / nb
    return np.array(alphas), np.array(betas)


def quadrature(alphas, betas):
    """sum tau_1i^2 log(lambda_i) of the tridiagonal, solvers.py:155-161."""
    lam, vec = scipy.linalg.eigh_tridiagonal(alphas, betas)
    if lam.min() <= 0.0:
        raise OracleNotSpd(f"nonpositive Ritz value {lam.min():g}")
    tau = vec[0]
    return float(np.sum(tau * tau * np.log(lam)))


def probes(n, count, seed=0):
    """Rademacher probes of slq_logdet, solvers.py:175-177 (prefix-stable)."""
    out = np.empty((n, count))
    for c, child in enumerate(np.random.SeedSequence(seed).spawn(count)):
        rng = np.random.Generator(np.random.PCG64(child))
        out[:, c] = rng.integers(0, 2, size=n) * 2.0 - 1.0
    return out


def slq_logdet(apply, n, probes_count=16, steps=50, seed=0):
    """Mean over probes of n * quadrature, solvers.py:164-179."""
    steps = min(steps, n)
    z = probes(n, probes_count, seed)
    total = 0.0
    for c in range(probes_count):
        a, b = lanczos(apply, np.ascontiguousarray(z[:, c]), steps)
        total += n * quadrature(a, b)
    return total / probes_count


# ------------------------------------------------------------------ model layer

DENSE_OPERATOR_MAX = 2048  # models.py:44
CG_FIT_BLOCK = 32  # models.py:45
FIT_CG_TOLERANCE = 1e-8  # models.py:46


def operator(nodes, x, noise):
    """The CG operator gp_fit builds, models.py:174-189 / _operator :203-213."""
    n = x.shape[0]
    if n <= DENSE_OPERATOR_MAX:
        g = gram(nodes, x, x, same=True)
        g.flat[:: n + 1] += noise
        return lambda v: g @ v
    return lambda v: matvec(nodes, x, noise, v, block=CG_FIT_BLOCK)


def fit(nodes, x, y, noise, rel_tol=FIT_CG_TOLERANCE, max_iter=None):
    """gp_fit(..., 'cg') -> (alpha, iterations, residual); models.py:143-189."""
    return cg(operator(nodes, x, noise), y, rel_tol, max_iter)


def predict(nodes, x, noise, alpha, xs, rel_tol=FIT_CG_TOLERANCE, max_iter=None):
    """gp_predict CG branch, models.py:216-250 -> (mean, var)."""
    kstar = gram(nodes, x, xs)
    mean = kstar.T @ alpha
    prior = diag(nodes, xs)
    app = operator(nodes, x, noise)
    quad = np.empty(xs.shape[0])
    for j in range(xs.shape[0]):
        col = kstar[:, j]  # strided view, as models.py:243 (affects dot rounding)
        sol = cg(app, col, rel_tol, max_iter)[0]
        quad[j] = col @ sol
    var = prior - quad
    np.maximum(var, 0.0, out=var)
    return mean, var


def lml(nodes, x, y, noise, alpha, probes_count=16, steps=50, seed=0):
    """log_marginal_likelihood CG branch, models.py:253-266."""
    n = y.shape[0]
    quad = float(y @ alpha)
    ld = slq_logdet(operator(nodes, x, noise), n, probes_count, steps, seed)
    return -0.5 * (quad + ld + n * LOG_2PI)


# -------------------------------------------------------------- synthetic inputs

CONFIGS = {
    # SURVEY.md §8(d) recipe; kernels as s-expressions (models use them verbatim)
    "cfg1": dict(kernel="(rbf 0.2)", n=2048, d=1, noise=0.01, t=1),
    "cfg2": dict(kernel="(matern52 0.5)", n=20000, d=4, noise=0.1, t=1),
    "cfg3": dict(kernel="(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))",
                 n=50000, d=2, noise=0.1, t=16),
    "cfg4": dict(kernel="(rbf 0.5)", n=100000, d=8, noise=0.1, t=16),
    "cfg5": dict(kernel="(matern32 0.5)", n=500000, d=8, noise=0.1, t=8),
}


def synthetic(n, d, seed=0):
    """X ~ U[0,1]^D (sorted for D=1), y = sin(2 pi sum(X)/sqrt(D)) + 0.1 eps."""
    rng = np.random.default_rng(seed)
    if d == 1:
        x = np.sort(rng.random(n))[:, None]
    else:
        x = rng.random((n, d))
    y = np.sin(2.0 * np.pi * x.sum(1) / math.sqrt(d)) + 0.1 * rng.standard_normal(n)
    return np.ascontiguousarray(x), np.ascontiguousarray(y)
