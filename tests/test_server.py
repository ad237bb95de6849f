"""The JSON-lines server over the device GP path (reference server.py and its
tests, test_server.py): protocol, error kinds and handle lifetime on the CPU;
fit / predict through the device CG on the GPU against the reference server's
own replies (tests/golden/make_server_golden.py)."""

import base64
import io
import json

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import golden
from paper_2605_17898_b200.server import Server, main


def encode(arr):
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    return {"shape": list(arr.shape), "data": base64.b64encode(arr.tobytes()).decode()}


def decode(obj):
    return np.frombuffer(base64.b64decode(obj["data"]), dtype="<f8").reshape(obj["shape"])


def step(server, **request):
    return server.step(json.dumps(request))


def make_data(seed=0, n=50):
    rng = np.random.default_rng(seed)
    x = rng.random((n, 2))
    y = np.sin(3.0 * x[:, 0]) + 0.1 * rng.standard_normal(n)
    return x, y


# ------------------------------------------------------------------ CPU side

def test_ping_and_id_echo():
    reply = step(Server(), id=1, op="ping")
    assert reply["ok"] and reply["result"]["version"] == G.__version__
    assert reply["id"] == 1


def test_metrics_op_matches_reference_replies_bitwise():
    g = golden("server.npz")
    server = Server()
    for c in range(3):
        mean, var, y = g[f"m{c}_in"]
        reply = step(server, id=c, op="metrics", mean=encode(mean), variance=encode(var),
                     y_true=encode(y), noise=0.1 * (c + 1))
        r = reply["result"]
        assert [r["rmse"], r["nll"], r["coverage95"]] == list(g[f"m{c}_out"])
        assert G.metrics(mean, var, 0.1 * (c + 1), y) == tuple(g[f"m{c}_out"])


def test_error_kinds_before_the_device():
    server = Server()
    x, y = make_data()
    assert step(server, id=1, op="fit", kernel="(rbf oops)", noise=0.1, x=encode(x),
                y=encode(y))["error"]["kind"] == "parse"
    assert step(server, id=2, op="fit", kernel="(rbf 0.5)", noise=0.1, x=encode(x),
                y=encode(y[:10]))["error"]["kind"] == "shape"
    assert step(server, id=3, op="fit", kernel="(rbf 0.5)", noise=0.1, x=encode(x),
                y=encode(y.reshape(10, 5)))["error"]["kind"] == "shape"
    bad = encode(x)
    bad["shape"] = [20, 2]  # shape disagrees with the payload
    assert step(server, id=4, op="fit", kernel="(rbf 0.5)", noise=0.1, x=bad,
                y=encode(y))["error"]["kind"] == "shape"
    nan = y.copy()
    nan[3] = np.nan
    assert step(server, id=5, op="fit", kernel="(rbf 0.5)", noise=0.1, x=encode(x),
                y=encode(nan))["error"]["kind"] == "shape"
    assert step(server, id=6, op="fit", kernel="(rbf 0.5)", noise=0.0, x=encode(x),
                y=encode(y))["error"]["kind"] == "shape"  # noise must be positive
    assert step(server, id=7, op="predict", handle=99, x=encode(x))["error"]["kind"] == "disposed"
    assert step(server, id=8, op="launch")["error"]["kind"] == "shape"
    reply = server.step("{not json")
    assert not reply["ok"] and reply["error"]["kind"] == "parse" and reply["id"] is None
    assert step(server, id=9, op="dispose", handle=123)["result"] == {"disposed": True}
    assert step(server, id=10, op="ping")["ok"]  # still up


def test_main_loop_one_reply_per_line():
    out = io.StringIO()
    lines = [json.dumps({"id": 1, "op": "ping"}), "", "{bad", json.dumps({"id": 2, "op": "nope"})]
    assert main(io.StringIO("\n".join(lines) + "\n"), out) == 0
    replies = [json.loads(s) for s in out.getvalue().splitlines()]
    assert [r["ok"] for r in replies] == [True, False, False]
    assert [r["id"] for r in replies] == [1, None, 2]


# ------------------------------------------------------------------ GPU side

@pytest.mark.gpu
def test_fit_predict_device_matches_core_and_reference(gpu_ctx):
    g = golden("server.npz")
    server = Server()
    x, y, xs = g["fit_x"], g["fit_y"], g["fit_xs"]
    fit = step(server, id=1, op="fit", kernel="(rbf 0.4)", noise=0.05, x=encode(x), y=encode(y))
    assert fit["ok"], fit
    pred = step(server, id=2, op="predict", handle=fit["result"]["handle"], x=encode(xs))
    mean, var = decode(pred["result"]["mean"]), decode(pred["result"]["variance"])
    # the same calls through the Python API give the same bits
    st = G.gp_fit(x, y, G.RBF(0.4), 0.05, "cg")
    m2, v2 = G.gp_predict(st, xs)
    np.testing.assert_array_equal(mean, m2)
    np.testing.assert_array_equal(var, v2)
    # and the reference server's replies within the north star's bars
    assert np.linalg.norm(mean - g["fit_mean"]) <= 1e-4 * np.linalg.norm(g["fit_mean"])
    assert np.max(np.abs(var - g["fit_var"])) <= 3e-3


@pytest.mark.gpu
def test_handles_empty_sets_and_dispose(gpu_ctx):
    server = Server()
    xa, ya = make_data(seed=3)
    xb, yb = make_data(seed=4)
    ha = step(server, id=1, op="fit", kernel="(rbf 0.4)", noise=0.05, x=encode(xa),
              y=encode(ya))["result"]["handle"]
    hb = step(server, id=2, op="fit", kernel="(rbf 0.4)", noise=0.05, x=encode(xb),
              y=encode(yb))["result"]["handle"]
    assert ha != hb
    xs = np.random.default_rng(5).random((4, 2))
    pa = decode(step(server, id=3, op="predict", handle=ha, x=encode(xs))["result"]["mean"])
    pb = decode(step(server, id=4, op="predict", handle=hb, x=encode(xs))["result"]["mean"])
    assert not np.array_equal(pa, pb)
    empty = step(server, id=5, op="predict", handle=ha, x=encode(np.empty((0, 2))))["result"]
    assert empty["mean"]["shape"] == [0] and empty["variance"]["shape"] == [0]
    assert step(server, id=6, op="dispose", handle=ha)["result"]["disposed"]
    assert step(server, id=7, op="predict", handle=ha, x=encode(xs))["error"]["kind"] == "disposed"
    assert step(server, id=8, op="dispose", handle=ha)["ok"]  # idempotent
    pb2 = decode(step(server, id=9, op="predict", handle=hb, x=encode(xs))["result"]["mean"])
    np.testing.assert_array_equal(pb, pb2)
