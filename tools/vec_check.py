"""Pinned-budget CG: the one-launch vector step vs the 3-kernel step vs the FP64 oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
rng = np.random.default_rng(21)
x, b = rng.random((800, 4)), rng.standard_normal(800)
k = G.Matern52(0.5)
nodes = O.parse_tree(G.format_kernel(k))
for it in (1, 2, 5, 25):
    cfg = G.CgConfig(rel_tolerance=1e-30, max_iterations=it)
    ref = O.cg(lambda v: O.matvec(nodes, x, 0.1, v), b, 1e-30, it)
    out = {}
    for mode in ("vec1", "vec3", "unfused"):
        os.environ.pop("LGP_CG_VEC3", None); os.environ.pop("LGP_CG_UNFUSED", None)
        if mode == "vec3": os.environ["LGP_CG_VEC3"] = "1"
        if mode == "unfused": os.environ["LGP_CG_UNFUSED"] = "1"
        res = G.cg_solve(G.KernelOperator(k, x, 0.1), b, cfg)
        out[mode] = res.x
        print(it, mode, "relL2 vs oracle %.2e" % (np.linalg.norm(res.x - ref[0]) / np.linalg.norm(ref[0])), "res %.4e" % res.final_residual)
    print("  vec1 vs vec3 max diff", np.abs(out["vec1"] - out["vec3"]).max())
