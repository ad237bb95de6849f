"""Host-side profile of the public matvec call (pageable NumPy inputs, warm)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
cfg = O.CONFIGS["cfg4"]
x, _ = O.synthetic(cfg["n"], cfg["d"])
z = np.ascontiguousarray(O.probes(cfg["n"], 16))
k = G.parse_kernel(cfg["kernel"])
for _ in range(30):
    G.matrix_free_matvec(k, x, 0.1, z)
t0 = time.perf_counter()
for _ in range(20):
    G.matrix_free_matvec(k, x, 0.1, z)
print("per call %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    G.matrix_free_matvec(k, x, 0.1, z)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
