"""Generate golden fixtures from the REAL reference (minigp) — run in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference lives only in the build container (``/root/reference``); the GPU
box never sees it, so its outputs are frozen here as small ``.npz`` files.
Inputs are NOT stored: every case records the seed recipe (``inputs()``
below and ``oracle.gp_oracle.synthetic``), which NumPy's PCG64 reproduces
bit-for-bit on any platform; a checksum of each regenerated input is stored
to catch drift.

Fixtures
--------
matvec_small.npz   matrix_free_matvec on 300-point sets, 12 kernel trees
matvec_rows.npz    full-size cfg1..cfg5 inputs, output rows of the reference
                   loop body (solvers.py:79-80) for a row subset, t=1 and probes
cg_small.npz       cg_solve on the matrix-free operator (solvers.py:87-123)
slq_small.npz      slq_logdet + the per-probe Lanczos tridiagonals
model_cfg1.npz     gp_fit/gp_predict/log_marginal_likelihood, cfg1 in full
model_small.npz    the same on N=3000 (matrix-free branch) for cfg2..cfg5 kernels
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
import time

import numpy as np
import scipy.linalg

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import minigp as M  # noqa: E402  (reference, build container only)
import minigp.solvers as MS  # noqa: E402

from oracle import gp_oracle as O  # noqa: E402  (for the shared input recipe only)

SMALL_TREES = [
    "(rbf 0.5)",
    "(matern12 0.3)",
    "(matern32 0.4)",
    "(matern52 0.5)",
    "(periodic 0.8 1.3)",
    "(linear 0.7)",
    "(scale 1.5 (rbf 0.6))",
    "(+ (scale 2.0 (matern32 0.4)) (linear 0.5))",
    "(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))",
    "(* (rbf 0.5) (periodic 1.0 0.5))",
    "(* (scale 0.7 (matern52 0.9)) (+ (matern12 1.1) (rbf 0.3)))",
    "(+ (scale 0.5 (periodic 0.6 0.7)) (* (linear 0.2) (matern32 2.0)))",
]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def inputs(n, d, seed):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    v = rng.standard_normal(n)
    return x, v


def make_matvec_small():
    out = {}
    for ci, s in enumerate(SMALL_TREES):
        for d in (1, 3, 8):
            seed = 100 + ci * 10 + d
            x, v = inputs(300, d, seed)
            k = M.parse_kernel(s)
            y = M.matrix_free_matvec(k, x, 0.1, v, block=32)
            key = f"{ci}_{d}"
            out[f"y_{key}"] = y
            out[f"seed_{key}"] = seed
            out[f"tree_{key}"] = s
            out[f"xsha_{key}"] = digest(x)
    # multi-RHS: the 8 SLQ probes (solvers.py:175-177) as the right-hand sides
    x, _ = inputs(257, 4, 7)
    z = O.probes(257, 8, seed=3)
    k = M.parse_kernel("(matern52 0.5)")
    out["probe_y"] = np.stack([M.matrix_free_matvec(k, x, 0.25, np.ascontiguousarray(z[:, c]))
                               for c in range(8)], axis=1)
    out["probe_z"] = z
    np.savez_compressed(os.path.join(HERE, "matvec_small.npz"), **out)


ROW_SUBSETS = {"cfg1": (0, 256), "cfg2": (9000, 9256), "cfg3": (25000, 25128),
               "cfg4": (50000, 50128), "cfg5": (250000, 250064)}


def make_matvec_rows():
    out = {}
    for name, cfg in O.CONFIGS.items():
        t0 = time.time()
        x, _ = O.synthetic(cfg["n"], cfg["d"], seed=0)
        v = np.random.default_rng(1).standard_normal(cfg["n"])
        z = O.probes(cfg["n"], cfg["t"], seed=0) if cfg["t"] > 1 else None
        k = M.parse_kernel(cfg["kernel"])
        r0, r1 = ROW_SUBSETS[name]
        slab = k._gram(x[r0:r1], x)  # the reference loop body, solvers.py:79-80
        y1 = np.dot(slab, v) + cfg["noise"] * v[r0:r1]
        out[f"{name}_rows"] = np.array([r0, r1])
        out[f"{name}_y1"] = y1
        out[f"{name}_xsha"] = digest(x)
        if z is not None:
            yz = np.stack([np.dot(slab, np.ascontiguousarray(z[:, c])) for c in range(z.shape[1])], 1)
            yz += cfg["noise"] * z[r0:r1]
            out[f"{name}_yz"] = yz
        del slab
        print(name, f"{time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "matvec_rows.npz"), **out)


def make_cg_small():
    out = {}
    cases = [("(scale 1.2 (rbf 0.4))", 600, 2, 1e-8), ("(matern52 0.5)", 500, 4, 1e-8),
             ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 400, 2, 1e-6),
             ("(rbf 0.5)", 700, 8, 1e-10)]
    for ci, (s, n, d, tol) in enumerate(cases):
        x, b = inputs(n, d, 500 + ci)
        k = M.parse_kernel(s)
        res = M.cg_solve(lambda v: M.matrix_free_matvec(k, x, 0.1, v, block=32), b,
                         M.CgConfig(rel_tolerance=tol))
        out[f"x_{ci}"] = res.x
        out[f"it_{ci}"] = res.iterations
        out[f"res_{ci}"] = res.final_residual
        out[f"case_{ci}"] = np.array([n, d, 500 + ci])
        out[f"tree_{ci}"] = s
        out[f"tol_{ci}"] = tol
    np.savez_compressed(os.path.join(HERE, "cg_small.npz"), **out)


def make_slq_small():
    captured = []
    real = scipy.linalg.eigh_tridiagonal

    def spy(a, b, *args, **kw):
        captured.append((np.array(a), np.array(b)))
        return real(a, b, *args, **kw)

    out = {}
    cases = [("(scale 1.3 (matern32 0.5))", 300, 3, 6, 20, 0),
             ("(rbf 0.2)", 256, 1, 4, 50, 5)]
    MS.scipy.linalg.eigh_tridiagonal = spy
    try:
        for ci, (s, n, d, probes, steps, seed) in enumerate(cases):
            captured.clear()
            x, _ = inputs(n, d, 700 + ci)
            k = M.parse_kernel(s)
            ld = M.slq_logdet(lambda v: M.matrix_free_matvec(k, x, 0.1, v, block=32), n,
                              M.CgConfig(probes=probes, lanczos_steps=steps), seed=seed)
            out[f"logdet_{ci}"] = ld
            out[f"case_{ci}"] = np.array([n, d, 700 + ci, probes, steps, seed])
            out[f"tree_{ci}"] = s
            for p, (a, b) in enumerate(captured):
                out[f"alpha_{ci}_{p}"] = a
                out[f"beta_{ci}_{p}"] = b
    finally:
        MS.scipy.linalg.eigh_tridiagonal = real
    np.savez_compressed(os.path.join(HERE, "slq_small.npz"), **out)


def model_case(s, x, y, noise, xs):
    k = M.parse_kernel(s)
    t0 = time.time()
    st = M.gp_fit(x, y, k, noise, "cg")
    mean, var = M.gp_predict(st, xs)
    lml = M.log_marginal_likelihood(st, seed=0)
    print(s, x.shape, f"{time.time() - t0:.1f}s it={st.cg_iterations}", flush=True)
    return dict(alpha=st.alpha, it=st.cg_iterations, res=st.cg_final_residual,
                mean=mean, var=var, lml=lml)


def make_model_cfg1():
    cfg = O.CONFIGS["cfg1"]
    x, y = O.synthetic(cfg["n"], cfg["d"], seed=0)
    xs = np.linspace(0.0, 1.0, 101)[:, None]
    r = model_case(cfg["kernel"], x, y, cfg["noise"], xs)
    chol = M.gp_fit(x, y, M.parse_kernel(cfg["kernel"]), cfg["noise"], "cholesky")
    cm, cv = M.gp_predict(chol, xs)
    r.update(chol_mean=cm, chol_var=cv, chol_lml=M.log_marginal_likelihood(chol),
             xsha=digest(x))
    np.savez_compressed(os.path.join(HERE, "model_cfg1.npz"), **r)


def make_model_small():
    out = {}
    for name in ("cfg2", "cfg3", "cfg4", "cfg5"):
        cfg = O.CONFIGS[name]
        x, y = O.synthetic(3000, cfg["d"], seed=0)
        xs = np.random.default_rng(9).random((8, cfg["d"]))
        r = model_case(cfg["kernel"], x, y, cfg["noise"], xs)
        for key, val in r.items():
            out[f"{name}_{key}"] = val
        out[f"{name}_xsha"] = digest(x)
    np.savez_compressed(os.path.join(HERE, "model_small.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["matvec_small", "matvec_rows", "cg_small", "slq_small",
                             "model_cfg1", "model_small"]
    for w in which:
        t0 = time.time()
        globals()[f"make_{w}"]()
        print(f"== {w} {time.time() - t0:.1f}s", flush=True)
