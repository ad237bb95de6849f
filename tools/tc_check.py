"""Tensor-core K1 bring-up: parity vs the SIMT kernel and the oracle, then timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

ctx = _lib.default_context()
lib = _lib.lib()


def mv(expr, x, V, noise, flags):
    prog = G.kernels.program(G.parse_kernel(expr))
    pts = _lib.DevicePoints(ctx, x)
    V = np.ascontiguousarray(V)
    out = np.empty_like(V)
    _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, noise, _lib.vptr(V),
                              V.shape[1], _lib.vptr(out), flags))
    return out


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


rng = np.random.default_rng(0)
for expr, n, d, t in [("(rbf 0.5)", 300, 8, 16), ("(rbf 0.5)", 1000, 8, 16), ("(matern52 0.7)", 777, 4, 8),
                      ("(+ (scale 2.0 (rbf 0.4)) (scale 0.5 (matern32 0.9)))", 2049, 6, 20),
                      ("(scale 1.5 (matern32 0.5))", 4096, 8, 16)]:
    x = rng.random((n, d))
    V = rng.standard_normal((n, t))
    t0 = time.time()
    tc = mv(expr, x, V, 0.1, 0)
    dt = time.time() - t0
    simt = mv(expr, x, V, 0.1, _lib.FORCE_SIMT)
    ref = O.matvec(O.parse_tree(expr), x, 0.1, V)
    print(f"{expr:55s} n={n} d={d} t={t}: tc-vs-oracle {rel(tc, ref):.2e}  simt-vs-oracle {rel(simt, ref):.2e}  ({dt:.2f}s)", flush=True)

cfg = O.CONFIGS["cfg4"]
x, _ = O.synthetic(cfg["n"], cfg["d"])
z = np.ascontiguousarray(O.probes(cfg["n"], 16))
prog = G.kernels.program(G.parse_kernel(cfg["kernel"]))
pts = _lib.DevicePoints(ctx, x)
dv, do = C.c_void_p(), C.c_void_p()
_lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(dv)))
_lib.check(lib.lgp_device_alloc(ctx.handle, z.nbytes, C.byref(do)))
_lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(z), z.nbytes))
ctx.set_profile(True)
for flags in (0, _lib.FORCE_SIMT):
    for _ in range(3):
        _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, cfg["noise"], dv, 16,
                                  do, _lib.DEVICE_PTRS | flags))
    ms, k = ctx.k1_profile()
    out = np.empty_like(z)
    _lib.check(lib.lgp_memcpy_d2h(ctx.handle, _lib.vptr(out), do, z.nbytes))
    r0 = 50000
    want = O.matvec(O.parse_tree(cfg["kernel"]), x, cfg["noise"], z, block=32, row_range=(r0, r0 + 128))
    print(f"cfg4 t=16 flags={flags}: K1 {ms / k:.3f} ms/launch, {cfg['n']**2*16/(ms/k*1e-3)/1e12:.2f} T entry*RHS/s, rows relL2 {rel(out[r0:r0+128], want):.2e}", flush=True)
