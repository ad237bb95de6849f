"""K1-TC-sym time per CG matvec vs the super-tile size R (LGP_TS_R), one
process per R (the choice is made once per operator)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 and sys.argv[1] == "--child":
    import numpy as np
    import paper_2605_17898_b200 as G
    from paper_2605_17898_b200 import _lib
    from oracle import gp_oracle as O
    cfg = O.CONFIGS[sys.argv[2]]
    x, _ = O.synthetic(cfg["n"], cfg["d"])
    ctx = _lib.default_context()
    op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"], ctx=ctx)
    v = np.random.default_rng(1).standard_normal(cfg["n"])
    op.matvec(v)
    ctx.set_profile(True)
    ctx.k1_profile(reset=True)
    reps = 10 if cfg["n"] <= 100000 else 3
    for _ in range(reps):
        op.matvec(v)
    ms, n = ctx.k1_profile()
    print(f"{sys.argv[2]} R={os.environ.get('LGP_TS_R', 'auto')}: {ms / n:.3f} ms", flush=True)
    sys.exit(0)
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg4"]
rs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto", "8", "12", "16", "24", "32", "48"]
for c in cfgs:
    for r in rs:
        env = dict(os.environ)
        if r != "auto":
            env["LGP_TS_R"] = r
        subprocess.run([sys.executable, __file__, "--child", c], env=env, check=False)
