"""Per-step host timing of matrix_free_matvec's body (cfg4, pinned X / V), medians of 30 calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from paper_2605_17898_b200.linalg import as_matrix, as_block, tracked
from paper_2605_17898_b200.kernels import slab_buffer_count
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
T = {}
def step(name, t0):
    t1 = time.perf_counter(); T.setdefault(name, []).append((t1 - t0) * 1e3); return t1
res = None
for it in range(60):
    t0 = time.perf_counter(); ts = t0
    xa = as_matrix(px, "X"); t0 = step("as_matrix", t0)
    va = as_block(pv, "v"); t0 = step("as_block", t0)
    slab_buffer_count(k); t0 = step("slab", t0)
    op = G.KernelOperator(k, xa, 0.1, _validated=True); t0 = step("operator", t0)
    r = op._matvec(va); t0 = step("matvec", t0)
    del op; t0 = step("del_op", t0)
    res = r; t0 = step("swap_res", t0)
    step("total", ts)
for kk, v in T.items():
    v = np.array(v[20:])
    print(f"{kk:10s} median {np.median(v):7.3f}  max {v.max():7.3f} ms")
