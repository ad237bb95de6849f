"""Predictive-variance multi-RHS CG: iterations and time, SIMT vs tensor-core K1 (LGP_CG_TC)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O
name = sys.argv[1]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = O.CONFIGS[name]
x, y = O.synthetic(cfg["n"], cfg["d"])
k = G.parse_kernel(cfg["kernel"])
st = G.gp_fit(x, y, k, cfg["noise"], "cg")
op = st.operator
xs = np.random.default_rng(9).random((T, cfg["d"]))
test = _lib.DevicePoints(op.ctx, xs)
lib = _lib.lib()
for rep in range(2):
    quad = np.empty(T); it = np.zeros(T, dtype=np.int32); res = np.zeros(T)
    t0 = time.perf_counter()
    _lib.check(lib.lgp_predict_quad(op.ctx.handle, op.prog.handle, op.points.handle, test.handle,
                                    st.noise, 1e-8, 0, _lib.dptr(quad), _lib.iptr(it), _lib.dptr(res)))
    dt = time.perf_counter() - t0
print(f"{name} T={T} LGP_CG_TC={os.environ.get('LGP_CG_TC', 'default')}: {dt:.3f} s, iterations max {it.max()} "
      f"median {int(np.median(it))}, quad[0:3] {quad[:3]}")
