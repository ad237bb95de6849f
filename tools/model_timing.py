"""End-to-end model calls at the BASELINE configs' full sizes: gp_fit (device
CG, tol 1e-8) + log_marginal_likelihood (device SLQ, 16 x 50) + gp_predict
(200 test points: mean by the cross matvec, variance by one multi-RHS CG)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]:
    cfg = O.CONFIGS[name]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    k = G.parse_kernel(cfg["kernel"])
    G.gp_fit(x[:2000], y[:2000], k, cfg["noise"], "cg")  # warm-up (JIT)
    t0 = time.perf_counter(); st = G.gp_fit(x, y, k, cfg["noise"], "cg"); t1 = time.perf_counter()
    lml = G.log_marginal_likelihood(st, seed=0); t2 = time.perf_counter()
    xs = np.random.default_rng(9).random((200, cfg["d"]))
    mean, var = G.gp_predict(st, xs); t3 = time.perf_counter()
    print(f"{name} N={cfg['n']}: fit {t1 - t0:.3f} s ({st.cg_iterations} it), LML {t2 - t1:.3f} s "
          f"({lml:.4f}), predict 200 {t3 - t2:.3f} s", flush=True)
