"""Low-D (D = 2, 3) r^2 trees on the tensor-core kernels vs the SIMT kernels:
time and accuracy (rows subset vs the FP64 oracle), t = 1 (CG matvec) and 16."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import ctypes as C
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O
lib = _lib.lib()
ctx = _lib.default_context()
for expr, d in [("(rbf 0.5)", 2), ("(rbf 0.3)", 3), ("(matern52 0.5)", 2), ("(matern32 0.4)", 3)]:
    n = 100000
    rng = np.random.default_rng(d)
    x = rng.random((n, d))
    prog = G.kernels.program(G.parse_kernel(expr))
    pts = _lib.DevicePoints(ctx, x)
    for t in (1, 16):
        V = rng.standard_normal((n, t))
        dv, do = C.c_void_p(), C.c_void_p()
        _lib.check(lib.lgp_device_alloc(ctx.handle, V.nbytes, C.byref(dv)))
        _lib.check(lib.lgp_device_alloc(ctx.handle, V.nbytes, C.byref(do)))
        _lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(V), V.nbytes))
        ctx.set_profile(True)
        for _ in range(3):
            _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, 0.1, dv, t, do, _lib.DEVICE_PTRS))
        ms, cnt = ctx.k1_profile(reset=True)
        out = np.empty((n, t))
        _lib.check(lib.lgp_memcpy_d2h(ctx.handle, _lib.vptr(out), do, out.nbytes)) if hasattr(lib, "lgp_memcpy_d2h") else None
        ref = O.matvec(O.parse_tree(expr), x, 0.1, V, block=2048, row_range=(0, 2048))
        err = np.linalg.norm(out[:2048] - ref) / np.linalg.norm(ref)
        print(f"{expr} D={d} t={t}: K1 {ms / cnt:.3f} ms, rows relL2 {err:.2e} (LOWD={os.environ.get('LGP_TC_LOWD')})", flush=True)
        lib.lgp_device_free(ctx.handle, dv); lib.lgp_device_free(ctx.handle, do)
