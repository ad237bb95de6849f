import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
g = np.load("tests/golden/tierc_cfg3.npz")
cfg = O.CONFIGS["cfg3"]
x, y = O.synthetic(cfg["n"], cfg["d"])
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"])
res = G.cg_solve(op, y, G.CgConfig(rel_tolerance=1e-30, max_iterations=int(g["it"])))
print("it", res.iterations, "x rel", np.linalg.norm(res.x - g["x"]) / np.linalg.norm(g["x"]), "res rel", abs(res.final_residual - float(g["res"])) / float(g["res"]))
z = G.probe_block(cfg["n"], int(g["probes"]), 0)
al, be, cnt = op.lanczos(z, int(g["steps"]))
for c in range(int(g["probes"])):
    m = int(cnt[c]); q = G.solvers.gauss_quadrature(al[c, :m], be[c, :m - 1])
    print(c, q, g["quads"][c], abs(q - g["quads"][c]) / abs(g["quads"][c]))
