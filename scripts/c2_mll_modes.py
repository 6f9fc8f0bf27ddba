"""C2 MLL in both operator precisions against the reference golden and the
exact (dense Cholesky, fp64, cuSOLVER) log marginal likelihood."""

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))

import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import kernels, likelihood, synthetic as syn  # noqa: E402
from conftest import load_golden  # noqa: E402


def exact_mll(model, X, y):
    import torch
    K = kernels.kernel_block_device(model, X, X, add_noise=True)
    L = torch.linalg.cholesky(K)
    del K
    yc = torch.from_numpy(y - model.mean).cuda()[:, None]
    a = torch.cholesky_solve(yc, L)
    quad = float((yc * a).sum())
    logdet = 2.0 * float(torch.log(torch.diagonal(L)).sum())
    n = X.shape[0]
    return -0.5 * quad - 0.5 * logdet - 0.5 * n * math.log(2 * math.pi), quad, logdet


def main():
    g = load_golden("c2_mll")
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(w.n, w.d, 0)
    y = syn.rff_target(X, seed=1)
    m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    print("reference:", float(g["value"]), int(g["iterations"]), "logdet", float(g["logdet"]), "quad", float(g["quad"]))
    for prec in ("fp64", "fp32"):
        t0 = time.perf_counter()
        r = gp.mll_value_and_grad(m, X, y, gp.plan_from_budget(w.n), gp.WorkerPool(),
                                  likelihood.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank,
                                                      precision=prec), 0)
        el = time.perf_counter() - t0
        ref = g["grad_vals"]
        got = np.array([r.gradients[str(k)] for k in g["grad_keys"]])
        print(f"{prec}: value {r.value!r} iters {r.diagnostics.iterations} logdet {r.diagnostics.logdet_estimate} "
              f"quad {r.diagnostics.quad_term} ({el:.1f}s); |dv|/|v| {abs(r.value - float(g['value'])) / abs(float(g['value'])):.2e}"
              f" grad err/max {np.abs(got - ref).max() / np.abs(ref).max():.2e}", flush=True)
    t0 = time.perf_counter()
    ex = exact_mll(m, X, y)
    print(f"exact: value {ex[0]!r} quad {ex[1]} logdet {ex[2]} ({time.perf_counter() - t0:.1f}s)")


if __name__ == "__main__":
    main()
