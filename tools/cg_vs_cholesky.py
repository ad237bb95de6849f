"""Device CG (KernelOperator) vs an FP64 Cholesky solve of the same Gram
(reference test_solvers.py:133-147 analog): max abs error per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.linalg
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
for seed, n, d in ((0, 300, 2), (1, 1000, 2), (2, 3000, 8)):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    y = rng.standard_normal(n)
    k = G.Scale(1.3, G.RBF(0.3))
    gram = O.gram(O.parse_tree(G.format_kernel(k)), x, x, same=True)
    gram.flat[:: n + 1] += 1.0
    want = scipy.linalg.cho_solve(scipy.linalg.cho_factor(gram), y)
    res = G.cg_solve(G.KernelOperator(k, x, 1.0), y, G.CgConfig(rel_tolerance=1e-11, max_iterations=5 * n))
    print(seed, n, d, res.iterations, "max abs err %.2e" % np.max(np.abs(res.x - want)),
          "rel %.2e" % (np.linalg.norm(res.x - want) / np.linalg.norm(want)))
