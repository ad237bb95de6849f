"""Randomised parity sweep of the fused matvec (all kernels / paths the
dispatcher can pick: SIMT, symmetric SIMT, K1-TC, K1-TC-sym) against the
oracle: random kernel trees over the full grammar (kernels.py:445-513),
random shapes (n, D, t) including ragged tiles, random point scales.
Seeded, so every run checks the same 48 cases. Bar: the north star's matvec
relative L2 1e-5."""

import numpy as np
import pytest

import paper_2605_17898_b200 as G
from conftest import rel_l2
from oracle import gp_oracle as O

pytestmark = pytest.mark.gpu

LEAVES = ("rbf", "matern12", "matern32", "matern52", "periodic", "linear")


def random_tree(rng, depth):
    if depth == 0 or rng.random() < 0.35:
        leaf = LEAVES[rng.integers(len(LEAVES))]
        ell = float(np.round(rng.uniform(0.2, 2.0), 3))
        if leaf == "periodic":
            return f"(periodic {ell} {float(np.round(rng.uniform(0.5, 2.0), 3))})"
        if leaf == "linear":
            return f"(linear {float(np.round(rng.uniform(0.1, 1.0), 3))})"
        return f"({leaf} {ell})"
    op = ("scale", "+", "*")[rng.integers(3)]
    if op == "scale":
        return f"(scale {float(np.round(rng.uniform(0.3, 3.0), 3))} {random_tree(rng, depth - 1)})"
    return f"({op} {random_tree(rng, depth - 1)} {random_tree(rng, depth - 1)})"


def cases():
    rng = np.random.default_rng(20261018)
    out = []
    for i in range(48):
        expr = random_tree(rng, 3)
        n = int(rng.choice([1, 7, 129, 700, 1500, 2049]))
        d = int(rng.integers(1, 13))
        t = int(rng.choice([1, 2, 8, 16, 17, 33]))
        scale = float(rng.choice([0.3, 1.0, 3.0]))
        out.append((i, expr, n, d, t, scale))
    return out


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"c{c[0]}")
def test_random_tree_matvec(gpu_ctx, case):
    i, expr, n, d, t, scale = case
    rng = np.random.default_rng(i)
    x = rng.random((n, d)) * scale
    v = rng.standard_normal((n, t)) if t > 1 else rng.standard_normal(n)
    k = G.parse_kernel(expr)
    got = G.matrix_free_matvec(k, x, 0.1, v)
    want = O.matvec(O.parse_tree(G.format_kernel(k)), x, 0.1, v)
    assert rel_l2(got, want) <= 1e-5, (expr, n, d, t, scale, rel_l2(got, want))
