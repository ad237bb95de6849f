"""Small CG / matvec / Lanczos calls for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
rng = np.random.default_rng(3)
x = rng.random((700, 8))
b = rng.standard_normal(700)
k = G.parse_kernel("(scale 1.2 (rbf 0.6))")
op = G.KernelOperator(k, x, 0.1)
r = G.cg_solve(op, b, G.CgConfig(rel_tolerance=1e-8, max_iterations=5))  # K1-TC-sym
V = rng.standard_normal((700, 16))
out = G.matrix_free_matvec(k, x, 0.1, V)  # K1-TC
al, be, cnt = op.lanczos(G.probe_block(700, 16, 0), 6)
print("ok", r.iterations, float(np.abs(out).max()), int(cnt[0]))
# round 2b paths: low-D tensor-core kernels, few-RHS API matvec (one pass of 8),
# 32 / 64 RHS passes, the staged host upload (needs >= 2 column segments)
for d, t in ((2, 16), (1, 5), (8, 32), (8, 64)):
    xs = rng.random((700, d))
    Vs = rng.standard_normal((700, t))
    o = G.matrix_free_matvec(k, xs, 0.1, Vs)
    print("ok", d, t, float(np.abs(o).max()))
xb = rng.random((20000, 8))
Vb = rng.standard_normal((20000, 16))
print("ok staged", float(np.abs(G.matrix_free_matvec(k, xb, 0.1, Vb)).max()))
opb = G.KernelOperator(k, xb, 0.1)
rb = G.cg_solve(opb, Vb[:, 0].copy(), G.CgConfig(rel_tolerance=1e-8, max_iterations=4))  # k_cg1_vec
print("ok cg", rb.iterations)
