"""cfg5 (Matern-3/2, N=500k, D=8, t=8): full-size matvec parity on golden rows + timings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "matvec_rows.npz"))
cfg = O.CONFIGS["cfg5"]
x, y = O.synthetic(cfg["n"], cfg["d"])
z = np.ascontiguousarray(O.probes(cfg["n"], cfg["t"]))
ctx = _lib.default_context(); lib = _lib.lib()
prog = G.kernels.program(G.parse_kernel(cfg["kernel"])); pts = _lib.DevicePoints(ctx, x)
dv, do = C.c_void_p(), C.c_void_p()
_lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(dv))); _lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(do)))
_lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(z), z.nbytes))
ctx.set_profile(True)
r0, r1 = (int(a) for a in g["cfg5_rows"])
for flags in (0, _lib.FORCE_SIMT):
    for _ in range(2):
        _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, cfg["noise"], dv, cfg["t"], do, _lib.DEVICE_PTRS | flags))
    ms, k = ctx.k1_profile()
    out = np.empty_like(z); _lib.check(lib.lgp_memcpy_d2h(ctx.handle, _lib.vptr(out), do, z.nbytes))
    err = np.linalg.norm(out[r0:r1] - g["cfg5_yz"]) / np.linalg.norm(g["cfg5_yz"])
    print(f"cfg5 t=8 flags={flags}: K1 {ms/k:.1f} ms/launch = {cfg['n']**2*cfg['t']/(ms/k*1e-3)/1e12:.2f} T entry*RHS/s; rows relL2 {err:.2e}", flush=True)
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
v1 = np.random.default_rng(1).standard_normal(cfg["n"])
out1 = op(v1)
err = np.linalg.norm(out1[r0:r1] - g["cfg5_y1"]) / np.linalg.norm(g["cfg5_y1"])
ms, k = ctx.k1_profile()
print(f"cfg5 t=1 (symmetric kernel): K1 {ms/k:.1f} ms; rows relL2 {err:.2e}", flush=True)
t0 = time.time(); xs, it, res = op.cg(y, 1e-8, 20)
ms, k = ctx.k1_profile()
print(f"cfg5 CG 20 iterations: {time.time()-t0:.2f} s ({ms/max(k,1):.1f} ms/matvec)", flush=True)
