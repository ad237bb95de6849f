"""K1-TC accuracy vs the FP32 accumulation group (LGP_TC_G): relative L2 vs the oracle on
cfg4 rows (golden) and a Gaussian-RHS block."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_17898_b200 as G
from oracle import gp_oracle as O
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "matvec_rows.npz"))
cfg = O.CONFIGS["cfg4"]
x, _ = O.synthetic(cfg["n"], cfg["d"])
z = O.probes(cfg["n"], 16)
op = G.KernelOperator(G.parse_kernel(cfg["kernel"]), x, cfg["noise"])
out = op(z)
r0, r1 = (int(a) for a in g["cfg4_rows"])
e1 = np.linalg.norm(out[r0:r1] - g["cfg4_yz"]) / np.linalg.norm(g["cfg4_yz"])
V = np.random.default_rng(3).standard_normal((cfg["n"], 16))
out2 = op(V)
want = O.matvec(O.parse_tree(cfg["kernel"]), x, cfg["noise"], V, block=32, row_range=(r0, r1))
e2 = np.linalg.norm(out2[r0:r1] - want) / np.linalg.norm(want)
print(f"G={os.environ.get('LGP_TC_G', '8')}: probes relL2 {e1:.2e}, gaussian relL2 {e2:.2e}")
