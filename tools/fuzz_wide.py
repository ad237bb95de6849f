"""One-off wide fuzz of the fused matvec vs the oracle (random trees / shapes / scales)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_fuzz import random_tree
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 7
count = int(sys.argv[2]) if len(sys.argv) > 2 else 150
rng = np.random.default_rng(seed)
worst, bad = 0.0, []
for i in range(count):
    expr = random_tree(rng, 3)
    n = int(rng.choice([1, 2, 63, 64, 65, 127, 128, 129, 500, 1000, 2049, 3000]))
    d = int(rng.integers(1, 13))
    t = int(rng.choice([1, 1, 3, 8, 16, 17, 24, 33]))
    scale = float(rng.choice([0.1, 0.5, 1.0, 2.0, 5.0]))
    r = np.random.default_rng(1000 + i)
    x = r.random((n, d)) * scale
    v = r.standard_normal((n, t)) if t > 1 else r.standard_normal(n)
    k = G.parse_kernel(expr)
    got = G.matrix_free_matvec(k, x, 0.1, v)
    want = O.matvec(O.parse_tree(G.format_kernel(k)), x, 0.1, v)
    e = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
    worst = max(worst, e)
    if not e <= 1e-5:
        bad.append((i, expr, n, d, t, scale, e))
print(f"seed {seed}: {count} cases, worst relL2 {worst:.2e}, failures {len(bad)}")
for b in bad[:20]:
    print("  FAIL", b)
