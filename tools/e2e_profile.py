"""Break down the public-API matvec call (e2e) into its host/device phases."""
import os, sys, time
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
ctx = _lib.default_context()
hx, hv = C.c_void_p(), C.c_void_p()
_lib.check(lib.lgp_host_alloc(x.nbytes, C.byref(hx)))
_lib.check(lib.lgp_host_alloc(z.nbytes, C.byref(hv)))
px = np.ctypeslib.as_array(C.cast(hx, C.POINTER(C.c_double)), shape=x.shape); px[...] = x
pv = np.ctypeslib.as_array(C.cast(hv, C.POINTER(C.c_double)), shape=z.shape); pv[...] = z
if "--pageable" in sys.argv:  # ordinary NumPy arrays, as the bench's e2e leg passes them
    px, pv = x.copy(), z.copy()
for _ in range(12):
    res = G.matrix_free_matvec(k, px, 0.1, pv)
T = {}
def tic(name, f):
    t0 = time.perf_counter(); r = f(); T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
for _ in range(5):
    xa = tic("as_matrix", lambda: G.as_matrix(px))
    va = tic("as_block", lambda: G.linalg.as_block(pv))
    prog = tic("program", lambda: G.kernels.program(k))
    pts = tic("points_upload", lambda: _lib.DevicePoints(ctx, xa))
    out = tic("result_buffer", lambda: _lib.result_buffer(va.shape))
    tic("lgp_matvec", lambda: _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, 0.1, _lib.vptr(va), 16, _lib.vptr(out), _lib.INPUTS_FINITE)))
    tic("points_free", lambda: pts.__del__())
    t0 = time.perf_counter(); G.matrix_free_matvec(k, px, 0.1, pv); T["full_call"] = T.get("full_call", 0) + time.perf_counter() - t0
for kk, v in T.items():
    print(f"{kk:15s} {v / 5 * 1e3:8.2f} ms")
