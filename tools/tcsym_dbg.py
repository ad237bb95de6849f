"""K1-TC-sym vs the SIMT kernel on one small case: matvec error split by row/column blocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
for n in (128, 256, 640, 3000):
    rng = np.random.default_rng(41)
    x = rng.random((n, 8))
    k = G.parse_kernel("(scale 1.2 (rbf 0.6))")
    v = np.random.default_rng(5).standard_normal(n)
    ref = O.matvec(O.parse_tree(G.format_kernel(k)), x, 0.1, v)
    op = G.KernelOperator(k, x, 0.1)
    out = op(v)
    err = np.abs(out - ref) / np.abs(ref).max()
    print(n, "relL2 %.3e" % (np.linalg.norm(out - ref) / np.linalg.norm(ref)),
          "worst rows", np.argsort(err)[-8:], "max %.3e" % err.max())
    if n == 128:
        # unit vectors: column j of the operator
        for j in (0, 1, 5, 64, 127):
            e = np.zeros(n); e[j] = 1
            o = op(e); r = O.matvec(O.parse_tree(G.format_kernel(k)), x, 0.1, e)
            bad = np.nonzero(np.abs(o - r) > 1e-5)[0]
            print("  e_%d bad rows" % j, bad[:20], len(bad))
