"""Wall time of optimize_hyperparams (exact-GP evidence objective) with the
2P+1 evaluations of a step run one by one vs concurrently (per-thread contexts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
for n in (600, 4000, 20000):
    rng = np.random.default_rng(17)
    x = rng.random((n, 3))
    y = np.sin(2.0 * x.sum(1)) + 0.1 * rng.standard_normal(n)
    kernel = G.parse_kernel("(scale 1.0 (rbf 0.5))")
    res = {}
    for workers in (1, 7):
        obj = G.exact_evidence_objective(x, y, kernel, seed=0, workers=workers)
        cfg = G.OptimizerConfig(steps=1, learning_rate=0.05)
        G.optimize_hyperparams(obj, G.flatten_model_params(kernel, 0.1), cfg)  # warm-up (JIT, contexts)
        cfg = G.OptimizerConfig(steps=3, learning_rate=0.05)
        t0 = time.perf_counter()
        best, trace = G.optimize_hyperparams(obj, G.flatten_model_params(kernel, 0.1), cfg)
        res[workers] = (time.perf_counter() - t0, trace)
    same = res[1][1] == res[7][1]
    print(f"N={n}: 3 Adam steps (21 evidence evaluations) sequential {res[1][0]:.3f} s, "
          f"7 concurrent contexts {res[7][0]:.3f} s, traces identical: {same}", flush=True)
