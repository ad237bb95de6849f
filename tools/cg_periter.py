"""Per-iteration wall time of the device CG at full size: two fixed budgets,
difference / extra iterations (removes per-call setup), next to the K1 time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

ctx = _lib.default_context()
for name in (sys.argv[1:] or ["cfg4"]):
    cfg = O.CONFIGS[name]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
    op.cg(y, 1e-30, 4)
    ts = {}
    for it in (100, 300):
        ctx.set_profile(True)
        ctx.k1_profile(reset=True)
        t0 = time.perf_counter()
        op.cg(y, 1e-30, it)
        ts[it] = time.perf_counter() - t0
        ms, n = ctx.k1_profile()
    per = (ts[300] - ts[100]) / 200 * 1e3
    print(f"{name}: {per:.3f} ms per CG iteration, K1 {ms / n:.3f} ms -> {1e3 * (per - ms / n):.1f} us "
          f"of other work per iteration; setup ~{(ts[100] - 100 * per / 1e3) * 1e3:.1f} ms per call",
          flush=True)
