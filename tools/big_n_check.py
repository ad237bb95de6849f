"""t = 1 matvec at N = 700000 (K1-TC-sym partial records beyond the 16 GB base
budget): a row subset against the oracle, and the time per launch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 700000
x, _ = O.synthetic(n, 8)
k = G.parse_kernel("(rbf 0.5)")
ctx = _lib.default_context()
op = G.KernelOperator(k, x, 0.1, ctx=ctx)
v = np.random.default_rng(1).standard_normal(n)
out = op(v)
ctx.set_profile(True); ctx.k1_profile(reset=True)
t0 = time.perf_counter(); out = op(v); dt = time.perf_counter() - t0
ms, cnt = ctx.k1_profile()
want = O.matvec(O.parse_tree("(rbf 0.5)"), x, 0.1, v, block=64, row_range=(n // 2, n // 2 + 64))
err = np.linalg.norm(out[n // 2:n // 2 + 64] - want) / np.linalg.norm(want)
print(f"N={n}: K1 {ms / max(cnt, 1):.1f} ms/launch, call {dt * 1e3:.1f} ms, rows relL2 {err:.2e}, "
      f"src has tcsym: {'lgp_matvec_tcsym' in G.kernels.program(k).source(8, 16)}")
