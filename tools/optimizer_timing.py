"""Wall time of optimize_hyperparams (exact-GP evidence objective): the 2P+1
evaluations of a step one by one, concurrently on per-thread contexts, and
with shift fusion (points differing only in output scale / noise share one
multi-shift CG + one Lanczos run). python tools/optimizer_timing.py [N ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
for n in [int(a) for a in sys.argv[1:]] or [4000, 20000]:
    rng = np.random.default_rng(17)
    x = rng.random((n, 4))  # cfg2's dimension
    y = np.sin(2.0 * x.sum(1)) + 0.1 * rng.standard_normal(n)
    kernel = G.parse_kernel("(scale 1.0 (rbf 0.5))")
    res = {}
    for name, kw in (("sequential", dict(workers=1, fuse_shifts=False)),
                     ("7 contexts", dict(workers=7, fuse_shifts=False)),
                     ("fused + 3 contexts", dict(workers=3, fuse_shifts=True))):
        obj = G.exact_evidence_objective(x, y, kernel, seed=0, **kw)
        cfg = G.OptimizerConfig(steps=1, learning_rate=0.05)
        G.optimize_hyperparams(obj, G.flatten_model_params(kernel, 0.1), cfg)  # warm-up (JIT, contexts)
        cfg = G.OptimizerConfig(steps=3, learning_rate=0.05)
        t0 = time.perf_counter()
        best, trace = G.optimize_hyperparams(obj, G.flatten_model_params(kernel, 0.1), cfg)
        res[name] = (time.perf_counter() - t0, trace)
    ref = np.array(res["sequential"][1])
    line = ", ".join(f"{k} {v[0]:.3f} s (trace max rel diff {np.max(np.abs(np.array(v[1]) - ref) / np.abs(ref)):.1e})"
                     for k, v in res.items())
    print(f"N={n}: 3 Adam steps (21 evidence evaluations): {line}", flush=True)
