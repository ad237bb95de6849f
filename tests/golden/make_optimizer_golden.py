"""Golden values for the hyper-parameter optimiser, from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_optimizer_golden.py

optimizer.npz
  toy_*   optimize_hyperparams on a deterministic analytic objective (30 steps):
          best parameters, centre trace, evaluation count - pure host logic,
          reproduced bit for bit by the package.
  flat_*  flatten_model_params / unflatten_model_params of a composite kernel.
  gp_*    3 Adam steps on the exact-GP evidence of a 600-point D = 3 problem
          (reference: cg strategy, dense operator for N <= 2048, SLQ seed 0).
"""

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import minigp as M  # noqa: E402  (reference, build container only)
import minigp.models as MM  # noqa: E402


def toy(q):
    c = np.array([0.3, -1.2, 0.8])
    w = np.array([1.0, 0.5, 2.0])
    return float(-np.sum(w * (q - c) ** 2) + 0.1 * math.sin(3.0 * q[0]) - 0.05 * q[1] * q[2])


def main():
    out = {}
    cfg = MM.OptimizerConfig(steps=30, learning_rate=0.1)
    p0 = np.array([0.0, 0.0, 0.0])
    best, trace = MM.optimize_hyperparams(toy, p0, cfg)
    out.update(toy_best=best, toy_trace=np.array(trace), toy_evals=cfg.evaluations)
    k = M.parse_kernel("(+ (scale 1.3 (rbf 0.6)) (matern52 0.9))")
    flat = MM.flatten_model_params(k, 0.2)
    k2, noise2 = MM.unflatten_model_params(k, flat + 0.1)
    out.update(flat_values=flat, flat_kernel2=M.format_kernel(k2), flat_noise2=noise2)
    rng = np.random.default_rng(17)
    x = rng.random((600, 3))
    y = np.sin(2.0 * x.sum(1)) + 0.1 * rng.standard_normal(600)
    kernel = M.parse_kernel("(scale 1.0 (rbf 0.5))")

    def evidence(q):
        kq, nq = MM.unflatten_model_params(kernel, q)
        st = M.gp_fit(x, y, kq, nq, "cg")
        return M.log_marginal_likelihood(st, seed=0)

    gcfg = MM.OptimizerConfig(steps=3, learning_rate=0.05)
    gbest, gtrace = MM.optimize_hyperparams(evidence, MM.flatten_model_params(kernel, 0.1), gcfg)
    out.update(gp_best=gbest, gp_trace=np.array(gtrace), gp_evals=gcfg.evaluations)
    np.savez_compressed(os.path.join(HERE, "optimizer.npz"), **out)
    print({k: (v if np.ndim(v) == 0 else np.asarray(v).tolist()) for k, v in out.items()})


if __name__ == "__main__":
    main()
