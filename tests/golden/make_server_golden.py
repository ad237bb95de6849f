"""Golden replies of the REFERENCE JSON server (minigp.server) for the port's
server tests. Build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_server_golden.py
"""

import base64
import json
import os

import numpy as np
from minigp.server import Server  # reference

HERE = os.path.dirname(os.path.abspath(__file__))


def enc(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return {"shape": list(a.shape), "data": base64.b64encode(a.tobytes()).decode()}


def dec(o):
    return np.frombuffer(base64.b64decode(o["data"]), dtype="<f8").reshape(o["shape"])


def main():
    out = {}
    s = Server()
    rng = np.random.default_rng(2)
    for c in range(3):
        mean, var, y = rng.standard_normal(9 + c), rng.random(9 + c), rng.standard_normal(9 + c)
        r = s.step(json.dumps({"id": c, "op": "metrics", "mean": enc(mean), "variance": enc(var),
                               "y_true": enc(y), "noise": 0.1 * (c + 1)}))["result"]
        out[f"m{c}_in"] = np.stack([mean, var, y])
        out[f"m{c}_out"] = np.array([r["rmse"], r["nll"], r["coverage95"]])
    # fit / predict through the reference's CG strategy (dense operator below N = 2049)
    rng = np.random.default_rng(0)
    x = rng.random((300, 2))
    y = np.sin(3.0 * x[:, 0]) + 0.1 * rng.standard_normal(300)
    xs = np.random.default_rng(1).random((7, 2))
    h = s.step(json.dumps({"id": 1, "op": "fit", "kernel": "(rbf 0.4)", "noise": 0.05,
                           "x": enc(x), "y": enc(y), "strategy": "cg"}))["result"]["handle"]
    p = s.step(json.dumps({"id": 2, "op": "predict", "handle": h, "x": enc(xs)}))["result"]
    out["fit_x"], out["fit_y"], out["fit_xs"] = x, y, xs
    out["fit_mean"], out["fit_var"] = dec(p["mean"]), dec(p["variance"])
    np.savez_compressed(os.path.join(HERE, "server.npz"), **out)
    print("wrote server.npz")


if __name__ == "__main__":
    main()
