"""K1 time for RBF + Periodic trees vs D (Periodic feature block PF = 2D per leaf):
tensor-core path (default) vs FORCE_SIMT, t = 1 and 16, N = 30000."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
ctx = _lib.default_context()
lib = _lib.lib()
n = 30000
for expr in ("(+ (rbf 0.5) (periodic 1.0 1.0))", "(+ (rbf 0.5) (* (periodic 1.0 1.0) (periodic 0.7 2.0)))"):
    for d in (2, 4, 8, 12):
        x = np.random.default_rng(d).random((n, d))
        prog = G.kernels.program(G.parse_kernel(expr))
        pts = _lib.DevicePoints(ctx, x)
        row = []
        for t in (1, 16):
            V = np.ascontiguousarray(np.random.default_rng(1).standard_normal((n, t)))
            dv, do = C.c_void_p(), C.c_void_p()
            _lib.check(lib.lgp_device_alloc(ctx.handle, V.nbytes, C.byref(dv)))
            _lib.check(lib.lgp_device_alloc(ctx.handle, V.nbytes, C.byref(do)))
            _lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(V), V.nbytes))
            for flags in (0, _lib.FORCE_SIMT):
                f = _lib.DEVICE_PTRS | flags
                _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, 0.1, dv, t, do, f))
                ctx.set_profile(True); ctx.k1_profile(reset=True)
                for _ in range(3):
                    _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, 0.1, dv, t, do, f))
                ms, k = ctx.k1_profile()
                row.append(f"t={t} {'simt' if flags else 'dflt'} {ms / k:.3f}")
        print(expr[:40], "d", d, " | ".join(row), flush=True)
