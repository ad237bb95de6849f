"""gp_predict's variance (one multi-RHS device CG over the T test points):
time, iteration distribution, vs the alpha solve. python tools/predict_timing.py cfg4 200"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = O.CONFIGS[name]
x, y = O.synthetic(cfg["n"], cfg["d"])
st = G.gp_fit(x, y, G.parse_kernel(cfg["kernel"]), cfg["noise"], "cg")
op = st.operator
xs = np.random.default_rng(9).random((T, cfg["d"]))
test = _lib.DevicePoints(op.ctx, xs)
lib = _lib.lib()
op.ctx.set_profile(True)
for rep in range(2):
    quad = np.empty(T); it = np.zeros(T, dtype=np.int32); res = np.zeros(T)
    op.ctx.k1_profile(reset=True)
    t0 = time.perf_counter()
    _lib.check(lib.lgp_predict_quad(op.ctx.handle, op.prog.handle, op.points.handle, test.handle,
                                    st.noise, 1e-8, 0, _lib.dptr(quad), _lib.iptr(it), _lib.dptr(res)))
    dt = time.perf_counter() - t0
    ms, n = op.ctx.k1_profile()
    if rep == 0:
        continue
    q = np.percentile(it, [0, 10, 50, 90, 100]).astype(int)
    print(f"{name} T={T}: {dt:.2f} s, alpha-solve iterations {st.cg_iterations}; variance CG "
          f"iterations min/p10/median/p90/max {q.tolist()}; K1 {ms / max(n, 1):.2f} ms x {n} launches",
          flush=True)
t0 = time.perf_counter()
mean, var = G.gp_predict(st, xs)
print(f"gp_predict({T}) {time.perf_counter() - t0:.2f} s", flush=True)
