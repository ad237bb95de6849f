"""Small driver for ncu: a few device-resident K1 launches at a config's full size."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--t", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
cfg = O.CONFIGS[a.config]
t = a.t or cfg["t"]
x, _ = O.synthetic(cfg["n"], cfg["d"])
z = np.ascontiguousarray(O.probes(cfg["n"], t))
ctx = _lib.default_context()
lib = _lib.lib()
prog = G.kernels.program(G.parse_kernel(cfg["kernel"]))
pts = _lib.DevicePoints(ctx, x)
dv, do = C.c_void_p(), C.c_void_p()
_lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(dv)))
_lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(do)))
_lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(z), z.nbytes))
ctx.set_profile(True)
for _ in range(a.reps):
    _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, cfg["noise"], dv, t, do,
                              _lib.DEVICE_PTRS | a.flags))
ms, n = ctx.k1_profile()
print(f"{a.config} t={t} flags={a.flags}: K1 {ms / n:.3f} ms/launch "
      f"({cfg['n'] ** 2 * t / (ms / n * 1e-3) / 1e12:.2f} T entry*RHS/s)")
