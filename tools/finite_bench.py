"""Input finiteness scan: threaded C (lgp_all_finite) vs NumPy, at the e2e V size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_17898_b200 import _lib
print("cpus", os.cpu_count())
for shape in ((100000, 16), (100000, 8), (500000, 8)):
    a = np.random.default_rng(0).standard_normal(shape)
    for name, f in (("C threads", lambda: _lib.all_finite(a)), ("numpy", lambda: bool(np.isfinite(a).all()))):
        f(); t0 = time.perf_counter()
        for _ in range(20): f()
        print(shape, name, f"{(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
