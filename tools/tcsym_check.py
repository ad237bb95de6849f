"""K1-TC-sym (super-tile, O(N) scratch) checks on the B200: single-RHS square
matvec parity vs the oracle over trees, ragged n and forced super-tile sizes
(LGP_TS_R), then cfg4 CG (iterations, time, K1 ms per matvec) and a cfg5-size
matvec. Usage: python tools/tcsym_check.py [--quick]"""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import paper_2605_17898_b200 as G
    from oracle import gp_oracle as O
    rng = np.random.default_rng(int(sys.argv[3]))
    worst = 0.0
    for s, d in [("(rbf 0.5)", 8), ("(matern32 0.5)", 8), ("(matern52 0.5)", 4),
                 ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 2)]:
        for n in (64, 129, 1000, 4097, 9000):
            x = rng.random((n, d))
            v = rng.standard_normal(n)
            got = G.matrix_free_matvec(G.parse_kernel(s), x, 0.1, v)
            want = O.matvec(O.parse_tree(s), x, 0.1, v, block=256)
            e = float(np.linalg.norm(got - want) / np.linalg.norm(want))
            again = G.matrix_free_matvec(G.parse_kernel(s), x, 0.1, v)
            assert np.array_equal(got, again), "not deterministic"
            worst = max(worst, e)
            if e > 1e-5:
                print("FAIL", s, n, e)
    print(f"R={os.environ.get('LGP_TS_R', 'auto')}: worst relL2 {worst:.2e}", flush=True)
    sys.exit(0)

for i, r in enumerate(["auto", "1", "2", "3", "8", "64"]):
    env = dict(os.environ)
    if r != "auto":
        env["LGP_TS_R"] = r
    subprocess.run([sys.executable, __file__, "--child", r, str(i)], env=env, check=True)
if len(sys.argv) > 1 and sys.argv[1] == "--quick":
    sys.exit(0)

import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O
ctx = _lib.default_context()
for name in ("cfg4", "cfg2", "cfg3"):
    cfg = O.CONFIGS[name]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
    op.cg(y, 1e-30, 2)
    ctx.set_profile(True)
    ctx.k1_profile(reset=True)
    t0 = time.perf_counter()
    xs, it, res = op.cg(y, 1e-8, None)
    dt = time.perf_counter() - t0
    ms, n = ctx.k1_profile()
    print(f"{name} CG to 1e-8: {int(it[0])} iterations, {dt:.3f} s, K1-TC-sym {ms / max(n, 1):.3f} ms x {n}",
          flush=True)
cfg = O.CONFIGS["cfg5"]
x, y = O.synthetic(cfg["n"], cfg["d"])
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
v = np.random.default_rng(1).standard_normal(cfg["n"])
out = op.matvec(v)
ctx.k1_profile(reset=True)
t0 = time.perf_counter()
out = op.matvec(v)
dt = time.perf_counter() - t0
ms, n = ctx.k1_profile()
r0 = 250000
want = O.matvec(O.parse_tree(cfg["kernel"]), x, cfg["noise"], v, block=32, row_range=(r0, r0 + 256))
e = float(np.linalg.norm(out[r0:r0 + 256] - want) / np.linalg.norm(want))
print(f"cfg5 t=1 matvec: K1-TC-sym {ms:.2f} ms, host call {dt * 1e3:.1f} ms, rows relL2 {e:.1e}", flush=True)
