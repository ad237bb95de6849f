"""SLQ log-det at a config's full size: phase timings (probes, device Lanczos, quadrature)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
cfg = O.CONFIGS[a.config]
x, y = O.synthetic(cfg["n"], cfg["d"])
n = cfg["n"]
t = cfg["t"] if cfg["t"] > 1 else 16
ctx = _lib.default_context()
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
op.lanczos(G.probe_block(n, t, 0), 2)
t0 = time.perf_counter(); z = G.probe_block(n, t, 0); t1 = time.perf_counter()
ctx.set_profile(True); ctx.k1_profile(reset=True)
al, be, cnt = op.lanczos(z, a.steps); t2 = time.perf_counter()
k1, nk = ctx.k1_profile(reset=True)
q = sum(G.solvers.gauss_quadrature(al[c, :cnt[c]], be[c, :cnt[c] - 1]) for c in range(t)); t3 = time.perf_counter()
print(f"probes {1e3*(t1-t0):.1f} ms, lanczos {1e3*(t2-t1):.1f} ms (K1 {k1:.1f} ms in {nk}), quadrature {1e3*(t3-t2):.1f} ms")
t0 = time.perf_counter(); ld = G.slq_logdet(op, n, G.CgConfig(probes=t, lanczos_steps=a.steps), seed=0)
print(f"slq_logdet total {1e3*(time.perf_counter()-t0):.1f} ms")
