"""Golden vectors for the training driver, by RUNNING THE REFERENCE
(blockgp 0.1.0 trainer.py) in the build container:

    python tests/golden/make_trainer_golden.py     # writes tests/golden/trainer.npz

1. Optimizer trajectories (adam_run, lbfgs_run) on a fixed analytic objective
   with a step-seeded perturbation, so the CPU tests pin the optimizer logic
   (moments, bias correction, two-loop recursion, Armijo backtracking, the
   shared-seed rule of one L-BFGS step) without a GPU.
2. A short full-adam training run on the C1 instance (n = 4,096, RBF):
   per-step MLL and the final raw parameters, for the GPU test.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import blockgp  # noqa: E402  (the reference)
from blockgp import trainer as rt  # noqa: E402
from make_golden import make_instance  # noqa: E402


class Bowl:
    """f(x) = sum w_i (x_i - c_i)^2 + 0.1 sum x_i^4 + 1e-3 (seed % 7) x_0:
    smooth, convex, and slightly different per probe seed."""

    def __init__(self, n, base_seed=3, fresh=True):
        self.w = np.linspace(1.0, 4.0, n)
        self.c = np.linspace(-1.0, 1.5, n)
        self.base_seed = base_seed
        self.fresh = fresh
        self.evals = 0

    def probe_seed(self, step):
        return self.base_seed + step if self.fresh else self.base_seed

    def __call__(self, x, step):
        self.evals += 1
        s = self.probe_seed(step) % 7
        f = float(np.sum(self.w * (x - self.c) ** 2) + 0.1 * np.sum(x ** 4) + 1e-3 * s * x[0])
        g = 2.0 * self.w * (x - self.c) + 0.4 * x ** 3
        g[0] += 1e-3 * s
        return f, g


def main():
    x0 = np.array([0.3, -0.7, 1.1, 0.0])
    xa, ta = rt.adam_run(Bowl(4), x0, rt.AdamConfig(lr=0.05, steps=25))
    xl, tl = rt.lbfgs_run(Bowl(4), x0, rt.LbfgsConfig(steps=8, history=3))
    out = dict(opt_x0=x0, adam_x=xa, adam_f=np.array([r.objective_value for r in ta.records]),
               adam_g=np.array([r.grad_norm for r in ta.records]), lbfgs_x=xl,
               lbfgs_f=np.array([r.objective_value for r in tl.records]),
               lbfgs_g=np.array([r.grad_norm for r in tl.records]))

    X, y, _ = make_instance(4096, 8)
    cfg = rt.TrainConfig(protocol="full-adam", family="rbf", adam=rt.AdamConfig(lr=0.1, steps=3), seed=0)
    model, trace = rt.train(X, y, cfg)
    out.update(c1_mll=np.array([r.mll for r in trace.records]),
               c1_iters=np.array([r.cg_iterations for r in trace.records]),
               c1_raw=blockgp.kernels.model_to_raw(model))
    path = os.path.join(HERE, "trainer.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: np.asarray(v).round(6).tolist() for k, v in out.items() if k.startswith("c1")})


if __name__ == "__main__":
    main()
