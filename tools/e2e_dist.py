"""Distribution of the public-API matvec wall time (cfg4, pinned X / V), 40 calls after warm-up."""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O
cfg = O.CONFIGS["cfg4"]
x, _ = O.synthetic(cfg["n"], cfg["d"])
z = np.ascontiguousarray(O.probes(cfg["n"], 16))
k = G.parse_kernel(cfg["kernel"])
lib = _lib.lib()
hx, hv = C.c_void_p(), C.c_void_p()
_lib.check(lib.lgp_host_alloc(x.nbytes, C.byref(hx)))
_lib.check(lib.lgp_host_alloc(z.nbytes, C.byref(hv)))
px = np.ctypeslib.as_array(C.cast(hx, C.POINTER(C.c_double)), shape=x.shape); px[...] = x
pv = np.ctypeslib.as_array(C.cast(hv, C.POINTER(C.c_double)), shape=z.shape); pv[...] = z
for _ in range(8):
    res = G.matrix_free_matvec(k, px, 0.1, pv)
ts = []
for _ in range(40):
    t0 = time.perf_counter(); res = G.matrix_free_matvec(k, px, 0.1, pv); ts.append((time.perf_counter() - t0) * 1e3)
ts = np.array(ts)
print("e2e ms: min %.2f median %.2f mean %.2f max %.2f" % (ts.min(), np.median(ts), ts.mean(), ts.max()))
print(" ".join(f"{t:.1f}" for t in ts))
