"""Device CG at a config's full size for a fixed number of iterations (ncu driver / timing)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
cfg = O.CONFIGS[a.config]
x, y = O.synthetic(cfg["n"], cfg["d"])
ctx = _lib.default_context()
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
op.cg(y, 1e-30, 2)  # warm-up (JIT, scratch)
ctx.set_profile(True)
ctx.k1_profile(reset=True)
t0 = time.perf_counter()
xs, iters, res = op.cg(y, 1e-30, a.iters)
dt = time.perf_counter() - t0
ms, n = ctx.k1_profile()
print(f"{a.config} CG {int(iters[0])} iterations: {dt * 1e3:.1f} ms wall, {dt * 1e3 / a.iters:.3f} ms/iter; "
      f"K1 {ms / max(n, 1):.3f} ms x {n}")
