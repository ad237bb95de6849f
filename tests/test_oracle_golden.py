"""Pins the CPU oracle to the real reference: every golden fixture made by
tests/golden/make_golden.py from minigp must be reproduced (bit-for-bit where
the operation order is identical)."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import gp_oracle as O


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def small_inputs(n, d, seed):
    rng = np.random.default_rng(seed)
    return rng.random((n, d)), rng.standard_normal(n)


def test_matvec_small_bitexact():
    g = golden("matvec_small.npz")
    keys = sorted(k[2:] for k in g.files if k.startswith("y_"))
    assert len(keys) == 36
    for key in keys:
        seed = int(g[f"seed_{key}"])
        d = int(key.split("_")[1])
        x, v = small_inputs(300, d, seed)
        assert digest(x) == str(g[f"xsha_{key}"])
        nodes = O.parse_tree(str(g[f"tree_{key}"]))
        got = O.matvec(nodes, x, 0.1, v, block=32)
        np.testing.assert_array_equal(got, g[f"y_{key}"])


def test_matvec_probe_block():
    g = golden("matvec_small.npz")
    x, _ = small_inputs(257, 4, 7)
    z = O.probes(257, 8, seed=3)
    np.testing.assert_array_equal(z, g["probe_z"])
    got = O.matvec(O.parse_tree("(matern52 0.5)"), x, 0.25, z, block=256)
    np.testing.assert_array_equal(got, g["probe_y"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_matvec_full_size_rows(name):
    g = golden("matvec_rows.npz")
    cfg = O.CONFIGS[name]
    x, _ = O.synthetic(cfg["n"], cfg["d"])
    assert digest(x) == str(g[f"{name}_xsha"])
    v = np.random.default_rng(1).standard_normal(cfg["n"])
    r0, r1 = (int(a) for a in g[f"{name}_rows"])
    nodes = O.parse_tree(cfg["kernel"])
    got = O.matvec(nodes, x, cfg["noise"], v, block=r1 - r0, row_range=(r0, r1))
    np.testing.assert_allclose(got, g[f"{name}_y1"], rtol=0, atol=1e-12 * np.abs(g[f"{name}_y1"]).max())
    if cfg["t"] > 1:
        z = O.probes(cfg["n"], cfg["t"])
        gz = O.matvec(nodes, x, cfg["noise"], z[:, :2], block=r1 - r0, row_range=(r0, r1))
        np.testing.assert_allclose(gz, g[f"{name}_yz"][:, :2], rtol=0,
                                   atol=1e-12 * np.abs(g[f"{name}_yz"]).max())


def test_cg_small():
    g = golden("cg_small.npz")
    for ci in range(4):
        n, d, seed = (int(a) for a in g[f"case_{ci}"])
        x, b = small_inputs(n, d, seed)
        nodes = O.parse_tree(str(g[f"tree_{ci}"]))
        sol, it, res = O.cg(lambda v: O.matvec(nodes, x, 0.1, v, block=32), b, float(g[f"tol_{ci}"]))
        assert it == int(g[f"it_{ci}"])
        np.testing.assert_array_equal(sol, g[f"x_{ci}"])
        assert res == float(g[f"res_{ci}"])


def test_slq_small():
    g = golden("slq_small.npz")
    for ci in range(2):
        n, d, seed, probes, steps, pseed = (int(a) for a in g[f"case_{ci}"])
        x, _ = small_inputs(n, d, seed)
        nodes = O.parse_tree(str(g[f"tree_{ci}"]))
        app = lambda v: O.matvec(nodes, x, 0.1, v, block=32)
        z = O.probes(n, probes, pseed)
        for p in range(probes):
            a, b = O.lanczos(app, np.ascontiguousarray(z[:, p]), min(steps, n))
            np.testing.assert_array_equal(a, g[f"alpha_{ci}_{p}"])
            np.testing.assert_array_equal(b, g[f"beta_{ci}_{p}"])
        ld = O.slq_logdet(app, n, probes, steps, pseed)
        assert ld == float(g[f"logdet_{ci}"])


def test_model_cfg1():
    g = golden("model_cfg1.npz")
    cfg = O.CONFIGS["cfg1"]
    x, y = O.synthetic(cfg["n"], cfg["d"])
    assert digest(x) == str(g["xsha"])
    nodes = O.parse_tree(cfg["kernel"])
    alpha, it, res = O.fit(nodes, x, y, cfg["noise"])
    assert it == int(g["it"])
    np.testing.assert_array_equal(alpha, g["alpha"])
    xs = np.linspace(0.0, 1.0, 101)[:, None]
    mean, var = O.predict(nodes, x, cfg["noise"], alpha, xs)
    np.testing.assert_array_equal(mean, g["mean"])
    np.testing.assert_array_equal(var, g["var"])
    lml = O.lml(nodes, x, y, cfg["noise"], alpha)
    assert lml == float(g["lml"])


def test_model_small_fit_cfg4_kernel():
    # matrix-free branch of gp_fit (N=3000 > 2048): the oracle reproduces the
    # reference's CG iterates bit for bit
    g = golden("model_small.npz")
    cfg = O.CONFIGS["cfg4"]
    x, y = O.synthetic(3000, cfg["d"])
    assert digest(x) == str(g["cfg4_xsha"])
    alpha, it, res = O.fit(O.parse_tree(cfg["kernel"]), x, y, cfg["noise"])
    assert it == int(g["cfg4_it"])
    np.testing.assert_array_equal(alpha, g["cfg4_alpha"])
