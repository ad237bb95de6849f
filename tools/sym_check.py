"""Symmetric block-pair K1: parity vs the plain kernel and the oracle, timing at cfg4 t=1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O

ctx = _lib.default_context(); lib = _lib.lib()
def mv(expr, x, V, noise, flags):
    prog = G.kernels.program(G.parse_kernel(expr)); pts = _lib.DevicePoints(ctx, x)
    V = np.ascontiguousarray(V); out = np.empty_like(V)
    _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, noise, _lib.vptr(V), V.shape[1], _lib.vptr(out), flags))
    return out
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
rng = np.random.default_rng(0)
for expr, n, d, t in [("(rbf 0.5)", 5000, 8, 1), ("(rbf 0.2)", 4100, 1, 1), ("(matern52 0.5)", 6000, 4, 4),
                      ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 4500, 2, 2)]:
    x = rng.random((n, d)); V = rng.standard_normal((n, t))
    a = mv(expr, x, V, 0.1, 0); b = mv(expr, x, V, 0.1, _lib.NO_SYM)
    ref = O.matvec(O.parse_tree(expr), x, 0.1, V, row_range=(0, 300))
    print(f"{expr:55s} n={n} t={t}: sym-vs-plain {rel(a, b):.2e} sym-vs-oracle(rows) {rel(a[:300], ref):.2e}", flush=True)
cfg = O.CONFIGS["cfg4"]
x, y = O.synthetic(cfg["n"], cfg["d"])
prog = G.kernels.program(G.parse_kernel(cfg["kernel"])); pts = _lib.DevicePoints(ctx, x)
v = np.ascontiguousarray(np.random.default_rng(1).standard_normal(cfg["n"]))
dv, do = C.c_void_p(), C.c_void_p()
_lib.check(lib.lgp_device_alloc(ctx.handle, v.nbytes, C.byref(dv))); _lib.check(lib.lgp_device_alloc(ctx.handle, v.nbytes, C.byref(do)))
_lib.check(lib.lgp_memcpy_h2d(ctx.handle, dv, _lib.vptr(v), v.nbytes))
ctx.set_profile(True)
for flags in (0, _lib.NO_SYM):
    for _ in range(3):
        _lib.check(lib.lgp_matvec(ctx.handle, prog.handle, pts.handle, pts.handle, 0.1, dv, 1, do, _lib.DEVICE_PTRS | flags))
    ms, k = ctx.k1_profile()
    print(f"cfg4 t=1 flags={flags}: K1 {ms/k:.3f} ms", flush=True)
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
t0 = time.time(); xs, it, res = op.cg(y, 1e-8, None); print(f"cfg4 CG: {time.time()-t0:.2f} s, {it[0]} iterations, res {res[0]:.3e}")
