"""Quick GPU sanity run: parity of the device path against the oracle + timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib
from oracle import gp_oracle as O


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


ctx = _lib.default_context()
rng = np.random.default_rng(0)
for s, n, d, t in [("(rbf 0.5)", 1000, 8, 1), ("(rbf 0.5)", 1000, 8, 16), ("(rbf 0.2)", 777, 1, 1),
                   ("(matern52 0.5)", 900, 4, 1), ("(matern12 0.3)", 500, 3, 2),
                   ("(+ (scale 1.0 (rbf 0.5)) (scale 1.0 (periodic 1.0 1.0)))", 700, 2, 16),
                   ("(matern32 0.5)", 1500, 8, 8), ("(+ (scale 2.0 (matern32 0.4)) (linear 0.5))", 300, 3, 3),
                   ("(periodic 0.1 1.0)", 400, 3, 4), ("(* (scale 0.7 (matern52 0.9)) (+ (matern12 1.1) (rbf 0.3)))", 333, 5, 5)]:
    x = rng.random((n, d))
    v = rng.standard_normal((n, t)) if t > 1 else rng.standard_normal(n)
    k = G.parse_kernel(s)
    t0 = time.time()
    got = G.matrix_free_matvec(k, x, 0.1, v)
    dt = time.time() - t0
    want = O.matvec(O.parse_tree(s), x, 0.1, v, block=256)
    g = G.kernel_eval(k, x)
    gw = O.gram(O.parse_tree(s), x, x, same=True)
    print(f"{s:60s} n={n} d={d} t={t} matvec relL2={rel(got, want):.2e} gram maxabs={np.abs(g-gw).max():.1e} sym={np.abs(g-g.T).max():.1e} ({dt:.2f}s)", flush=True)

# cfg4-size timing (device-resident via C ABI)
cfg = O.CONFIGS["cfg4"]
x, _ = O.synthetic(cfg["n"], cfg["d"])
z = O.probes(cfg["n"], 16)
k = G.parse_kernel(cfg["kernel"])
op = G.KernelOperator(k, x, cfg["noise"])
for t in (16, 1):
    V = np.ascontiguousarray(z[:, :t]) if t > 1 else np.ascontiguousarray(z[:, 0])
    op.matvec(V)
    ts = []
    for _ in range(3):
        t0 = time.time(); out = op.matvec(V); ts.append(time.time() - t0)
    print(f"cfg4 t={t} host-API matvec {min(ts)*1e3:.2f} ms -> {cfg['n']**2*t/min(ts)/1e9:.1f} Gentries/s", flush=True)
    r0, r1 = 50000, 50128
    want = O.matvec(O.parse_tree(cfg["kernel"]), x, cfg["noise"], V, block=32, row_range=(r0, r1))
    print("  rows parity relL2", rel(out[r0:r1], want), flush=True)
