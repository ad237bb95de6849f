"""CG iteration counts / solutions: symmetric SIMT K1 vs tensor-core K1 (LGP_CG_TC)."""
import os, sys, time, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
res = {}
for name, n in (("cfg4", 100000), ("cfg4", 20000), ("cfg2", 20000), ("cfg5", 50000)):
    cfg = O.CONFIGS[name]
    x, y = O.synthetic(n, cfg["d"])
    op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"])
    op.cg(y, 1e-8, 2)
    t0 = time.perf_counter(); xs, it, r = op.cg(y, 1e-8, None); dt = time.perf_counter() - t0
    res[f"{name}_{n}"] = (int(it[0]), float(r[0]), dt)
    np.save(f"/tmp/cgx_{name}_{n}_{os.environ.get('LGP_CG_TC', '0')}.npy", xs)
print(os.environ.get("LGP_CG_TC", "0"), json.dumps(res))
