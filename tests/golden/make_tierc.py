"""Full-size ("tier C") golden values from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tierc.py cfg2
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tierc.py cfg4
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tierc.py cfg3
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tierc.py n50k_rbf n50k_m32

Build container only (the reference is not on the GPU box).

fullsize_cfg2.npz  cfg2 in full (N = 20000, Matern-5/2, D = 4): the reference's own
                   cg_solve / slq_logdet / mean / LML code on the "dense replay"
                   operator (kernel_eval(X, X) + noise I, applied with dgemv: the
                   same kernel entries as matrix_free_matvec, only the summation
                   order of the matvec differs), plus the exact
                   (Cholesky) latent variance at 200 test points.
tierc_cfg4.npz     cfg4 in full (N = 100000, RBF, D = 8) through the reference's
                   real matrix_free_matvec (block = 32, the fit's block): CG after
                   exactly 20 iterations, and the SLQ quadratures of 16 probes
                   after 5 Lanczos steps (equal, pinned budgets; ~1.5 h of CPU).
tierc_n50k_rbf.npz / tierc_n50k_m32.npz
                   the cfg4 kernel (RBF 0.5, D = 8) and the cfg5 kernel (Matern-3/2
                   0.5, D = 8) at N = 50000 (the largest N whose FP64 Gram, 20 GB,
                   fits this container): the reference's own cg_solve (tol 1e-8) /
                   slq_logdet (16 probes x 50 steps) / mean / LML on the dense
                   replay operator built slab by slab from the reference's own
                   Kernel._gram (the entries matrix_free_matvec uses,
                   solvers.py:79-80), plus the exact (Cholesky) latent variance at
                   200 test points.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np
import scipy.linalg

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import minigp as M  # noqa: E402  (reference, build container only)
import minigp.solvers as MS  # noqa: E402

from oracle import gp_oracle as O  # noqa: E402  (shared input recipe only)


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def cfg2():
    cfg = O.CONFIGS["cfg2"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    n = x.shape[0]
    k = M.parse_kernel(cfg["kernel"])
    noise = cfg["noise"]
    log("cfg2 gram")
    gram_y = M.kernel_eval(k, x)
    gram_y.flat[:: n + 1] += noise
    apply = lambda v: gram_y @ v  # noqa: E731
    fit_cfg = M.CgConfig(rel_tolerance=1e-8)  # models.py FIT_CG_TOLERANCE
    log("cfg2 CG")
    res = M.cg_solve(apply, y, fit_cfg)
    log("cfg2 CG", res.iterations, res.final_residual)
    ld = M.slq_logdet(apply, n, fit_cfg, seed=0)
    quad = float(y @ res.x)
    lml = -0.5 * (quad + ld + n * np.log(2 * np.pi))
    log("cfg2 SLQ logdet", ld, "LML", lml)
    xs = np.random.default_rng(9).random((200, cfg["d"]))
    kstar = M.kernel_eval(k, x, xs)
    mean = kstar.T @ res.x
    log("cfg2 Cholesky")
    c = scipy.linalg.cho_factor(gram_y, lower=True, overwrite_a=False, check_finite=False)
    half = scipy.linalg.solve_triangular(c[0], kstar, lower=True, check_finite=False)
    var = np.maximum(M.kernel_diag(k, xs) - np.einsum("ij,ij->j", half, half), 0.0)
    chol_alpha = scipy.linalg.cho_solve(c, y, check_finite=False)
    np.savez_compressed(
        os.path.join(HERE, "fullsize_cfg2.npz"), it=res.iterations, res=res.final_residual,
        alpha=res.x, logdet=ld, lml=lml, mean=mean, var=var, chol_mean=kstar.T @ chol_alpha,
        note="reference cg_solve/slq_logdet on the dense replay operator; var by Cholesky")
    log("cfg2 done")


def cfg4():
    cfg = O.CONFIGS["cfg4"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    n = x.shape[0]
    k = M.parse_kernel(cfg["kernel"])
    noise = cfg["noise"]
    apply = lambda v: M.matrix_free_matvec(k, x, noise, v, block=32)  # noqa: E731
    it = 20
    log("cfg4 CG", it, "iterations")
    res = M.cg_solve(apply, y, M.CgConfig(rel_tolerance=1e-30, max_iterations=it))
    log("cfg4 CG", res.iterations, res.final_residual)
    np.savez_compressed(os.path.join(HERE, "tierc_cfg4_cg.npz"), it=res.iterations,
                        res=res.final_residual, x=res.x)
    steps, probes = 5, 16
    z = O.probes(n, probes, seed=0)
    quads = np.zeros(probes)
    for c in range(probes):
        quads[c] = MS._lanczos_quadrature(apply, np.ascontiguousarray(z[:, c]), steps)
        log("cfg4 probe", c, quads[c])
    np.savez_compressed(
        os.path.join(HERE, "tierc_cfg4.npz"), it=res.iterations, res=res.final_residual,
        x=res.x, steps=steps, probes=probes, quads=quads,
        note="reference matrix_free_matvec (block 32): CG after 20 iterations, "
             "per-probe Lanczos quadratures after 5 steps (probe seed 0)")
    log("cfg4 done")


def cfg3():
    # cfg3 (RBF + Periodic, N = 50000, D = 2): one reference matvec is ~3 min
    # here, so the pinned budgets are smaller: CG after 10 iterations, the
    # quadratures of 4 probes after 3 Lanczos steps (~22 reference matvecs)
    cfg = O.CONFIGS["cfg3"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    n = x.shape[0]
    k = M.parse_kernel(cfg["kernel"])
    noise = cfg["noise"]
    apply = lambda v: M.matrix_free_matvec(k, x, noise, v, block=32)  # noqa: E731
    it = 10
    log("cfg3 CG", it, "iterations")
    res = M.cg_solve(apply, y, M.CgConfig(rel_tolerance=1e-30, max_iterations=it))
    log("cfg3 CG", res.iterations, res.final_residual)
    steps, probes = 3, 4
    z = O.probes(n, probes, seed=0)
    quads = np.zeros(probes)
    for c in range(probes):
        quads[c] = MS._lanczos_quadrature(apply, np.ascontiguousarray(z[:, c]), steps)
        log("cfg3 probe", c, quads[c])
    np.savez_compressed(
        os.path.join(HERE, "tierc_cfg3.npz"), it=res.iterations, res=res.final_residual,
        x=res.x, steps=steps, probes=probes, quads=quads,
        note="reference matrix_free_matvec (block 32): CG after 10 iterations, "
             "per-probe Lanczos quadratures after 3 steps (probe seed 0)")
    log("cfg3 done")


def blocked_cholesky_solve_lower(a, rhs, nb=4096):
    """In place: the lower triangle of the symmetric `a` (C order) becomes L
    with a = L L^T (right-looking blocked Cholesky, every LAPACK / BLAS call on
    a block of < 2^31 elements); returns L^-1 rhs."""
    n = a.shape[0]
    for k0 in range(0, n, nb):
        k1 = min(n, k0 + nb)
        a[k0:k1, k0:k1] = scipy.linalg.cholesky(a[k0:k1, k0:k1], lower=True, check_finite=False)
        if k1 == n:
            break
        l11 = a[k0:k1, k0:k1]
        # panel below the diagonal block: A21 L11^-T
        a[k1:, k0:k1] = scipy.linalg.solve_triangular(l11, a[k1:, k0:k1].T, lower=True,
                                                      check_finite=False).T
        p = a[k1:, k0:k1]
        for j0 in range(k1, n, nb):  # trailing lower triangle, block column by block column
            j1 = min(n, j0 + nb)
            a[j0:, j0:j1] -= p[j0 - k1:] @ p[j0 - k1:j1 - k1].T
        log("  cholesky block", k0 // nb + 1, "of", -(-n // nb))
    h = np.empty_like(rhs)
    for k0 in range(0, n, nb):
        k1 = min(n, k0 + nb)
        t = rhs[k0:k1] - a[k0:k1, :k0] @ h[:k0]
        h[k0:k1] = scipy.linalg.solve_triangular(a[k0:k1, k0:k1], t, lower=True, check_finite=False)
    return h


def n50k(tag, scratch=os.environ.get("TIERC_SCRATCH", "/tmp/tierc")):
    # SURVEY.md §8c tier C: "check the same kernel/D/t at a reduced N where the
    # dense replay fits (N <= 50k)". Resumable: each stage's result is kept in
    # `scratch` (the CG, SLQ and Cholesky stages take minutes each).
    os.makedirs(scratch, exist_ok=True)
    kern = {"rbf": O.CONFIGS["cfg4"]["kernel"], "m32": O.CONFIGS["cfg5"]["kernel"]}[tag]
    n, d, noise = 50000, 8, 0.1
    x, y = O.synthetic(n, d)
    k = M.parse_kernel(kern)
    log(tag, "gram (slabs of the reference's _gram)")
    gram_y = np.empty((n, n))
    for i0 in range(0, n, 2048):
        i1 = min(n, i0 + 2048)
        gram_y[i0:i1] = k._gram(x[i0:i1], x)
    gram_y.flat[:: n + 1] += noise
    apply = lambda v: gram_y @ v  # noqa: E731
    fit_cfg = M.CgConfig(rel_tolerance=1e-8)  # models.py FIT_CG_TOLERANCE
    f_cg = os.path.join(scratch, f"{tag}_cg.npz")
    if not os.path.exists(f_cg):
        log(tag, "CG")
        res = M.cg_solve(apply, y, fit_cfg)
        np.savez(f_cg, it=res.iterations, res=res.final_residual, x=res.x)
    g = np.load(f_cg)
    it, resid, alpha = int(g["it"]), float(g["res"]), g["x"]
    log(tag, "CG", it, resid)
    f_slq = os.path.join(scratch, f"{tag}_slq.npz")
    if not os.path.exists(f_slq):
        ld = M.slq_logdet(apply, n, fit_cfg, seed=0)
        np.savez(f_slq, ld=ld)
    ld = float(np.load(f_slq)["ld"])
    quad = float(y @ alpha)
    lml = -0.5 * (quad + ld + n * np.log(2 * np.pi))
    log(tag, "SLQ logdet", ld, "LML", lml)
    xs = np.random.default_rng(9).random((200, d))
    kstar = M.kernel_eval(k, x, xs)
    mean = kstar.T @ alpha
    log(tag, "Cholesky (blocked: one LAPACK call on 50k^2 = 2.5e9 elements overflows the 32-bit "
             "indices of scipy's OpenBLAS)")
    half = blocked_cholesky_solve_lower(gram_y, kstar)
    var = np.maximum(M.kernel_diag(k, xs) - np.einsum("ij,ij->j", half, half), 0.0)
    np.savez_compressed(
        os.path.join(HERE, f"tierc_n50k_{tag}.npz"), kernel=kern, n=n, d=d, noise=noise,
        it=it, res=resid, alpha=alpha, logdet=ld, lml=lml, mean=mean,
        var=var, note="reference cg_solve/slq_logdet on the dense replay operator (slabs of "
                      "Kernel._gram); var by Cholesky")
    log(tag, "done")

if __name__ == "__main__":
    for name in sys.argv[1:]:
        {"cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4,
         "n50k_rbf": lambda: n50k("rbf"), "n50k_m32": lambda: n50k("m32")}[name]()
