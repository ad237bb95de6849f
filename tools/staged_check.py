"""The staged host-V upload (two parts, K1 per part) vs the one-copy path: results and e2e time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
for name in ("cfg4", "cfg3", "cfg2"):
    cfg = O.CONFIGS[name]
    x, _ = O.synthetic(cfg["n"], cfg["d"])
    z = np.ascontiguousarray(O.probes(cfg["n"], 16))
    k = G.parse_kernel(cfg["kernel"])
    out = {}
    for mode in ("staged", "plain"):
        if mode == "plain":
            os.environ["LGP_NO_STAGED"] = "1"
        else:
            os.environ.pop("LGP_NO_STAGED", None)
        for _ in range(10):
            r = G.matrix_free_matvec(k, x, cfg["noise"], z)
        t0 = time.perf_counter()
        for _ in range(20):
            r = G.matrix_free_matvec(k, x, cfg["noise"], z)
        dt = (time.perf_counter() - t0) / 20 * 1e3
        out[mode] = np.array(r)
        print(f"{name} {mode}: {dt:.3f} ms per call", flush=True)
    d = np.linalg.norm(out["staged"] - out["plain"]) / np.linalg.norm(out["plain"])
    print(f"  staged vs plain relL2 {d:.2e}")
