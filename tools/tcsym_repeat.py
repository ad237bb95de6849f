"""Repeatability of the symmetric tensor-core CG (same inputs -> same bits)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
rng = np.random.default_rng(43)
x = rng.random((2500, 2)); b = rng.standard_normal(2500)
k = G.parse_kernel("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))")
outs = []
for rep in range(4):
    r = G.cg_solve(G.KernelOperator(k, x, 0.1, ctx=_lib.Context(0)), b, G.CgConfig(rel_tolerance=1e-8))
    outs.append(r)
    print(rep, r.iterations, r.final_residual, float(np.abs(r.x - outs[0].x).max()), flush=True)
v = rng.standard_normal(2500)
op = G.KernelOperator(k, x, 0.1)
m = [op(v) for _ in range(5)]
print("matvec repeat max diff", max(float(np.abs(mm - m[0]).max()) for mm in m))
for R in ("1", "2", "4", "8"):
    os.environ["LGP_TS_R"] = R
    r = G.cg_solve(G.KernelOperator(k, x, 0.1, ctx=_lib.Context(0)), b, G.CgConfig(rel_tolerance=1e-8))
    print("R", R, r.iterations)
