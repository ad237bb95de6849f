import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
rng = np.random.default_rng(0)
for s, d in [("(rbf 0.5)", 8), ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 2), ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 4)]:
    for n in (300, 1000, 4097):
        x = rng.random((n, d)); v = rng.standard_normal(n)
        got = G.matrix_free_matvec(G.parse_kernel(s), x, 0.1, v)
        want = O.matvec(O.parse_tree(s), x, 0.1, v, block=256)
        print(os.environ.get("LGP_TS_NWG"), os.environ.get("LGP_TS_R"), s[:30], d, n, float(np.linalg.norm(got - want) / np.linalg.norm(want)), flush=True)
