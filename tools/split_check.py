"""Multi-rank (loopback) pair-split CG vs one rank at fixed budgets: the
iterates should agree to rounding (the all-reduce only reorders sums)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from paper_2605_17898_b200 import _lib


def run_ranks(world, fn):
    gid = b"LGP-LOOPBACK" + os.urandom(16)
    gid = gid + bytes(128 - len(gid))
    out = [None] * world
    def worker(r):
        ctx = _lib.Context(0, r, world, gid)
        try:
            out[r] = fn(ctx, r)
        finally:
            ctx.close()
    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    return out

rng = np.random.default_rng(5)
n, d = 2051, 5
x = rng.random((n, d))
b = rng.standard_normal(n)
k = G.parse_kernel("(+ (scale 1.1 (rbf 0.6)) (scale 0.4 (matern32 0.9)))")
for budget in (1, 2, 5, 20, 100, None):
    def fn(ctx, r):
        op = G.KernelOperator(k, x, 0.1, ctx=ctx)
        xs, it, res = op.cg(b, 1e-8 if budget is None else 1e-30, budget)
        return xs.copy(), int(it[0]), float(res[0])
    o2 = run_ranks(2, fn)[0]
    o1 = run_ranks(1, fn)[0]
    c1 = fn(_lib.default_context(), 0)  # plain single context (no communicator)
    e = np.linalg.norm(o2[0] - o1[0]) / np.linalg.norm(o1[0])
    e2 = np.linalg.norm(c1[0] - o1[0]) / np.linalg.norm(o1[0])
    print(f"budget {budget}: it {o2[1]} / {o1[1]} / {c1[1]}  relL2(world2 vs world1) {e:.2e}  (plain vs world1 {e2:.2e})", flush=True)
