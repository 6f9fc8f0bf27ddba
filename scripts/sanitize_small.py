"""Drive every kernel family of libgpbbmm once at small shapes, for
compute-sanitizer (tests/test_gpu_memory.py runs it under memcheck and
synccheck): K·V SIMT / row-tiled tcgen05 / symmetric / wide / large-d, mBCG,
pivoted Cholesky + Woodbury, MLL gradients (ARD and shared lengthscale),
prediction cache, mean and variance."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, likelihood, predictor  # noqa: E402

rng = np.random.default_rng(0)
for n, d, fam, t, algo in ((300, 5, "matern32", 11, 1), (300, 5, "rbf", 11, 2), (300, 5, "matern32", 11, 3),
                           (257, 3, "rbf", 16, 3), (300, 5, "matern32", 40, 0), (200, 50, "matern32", 11, 2)):
    X = rng.uniform(size=(n, d))
    m = gp.KernelModel(fam, 1.0, np.linspace(0.5, 1.5, d) * np.sqrt(d), 0.2)
    Xs32, _ = D.points(X).scaled(m.scale_for(d))
    op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.2, 0, algo=algo, self_offset=0)
    V = torch.from_numpy(rng.standard_normal((n, t))).float().cuda()
    op.apply32(V, t)
torch.cuda.synchronize()
print("kv ok", flush=True)
n, d = 400, 4
X = rng.uniform(size=(n, d))
y = rng.standard_normal(n)
for ard, fam in ((True, "matern32"), (False, "rbf")):
    ls = np.linspace(0.4, 0.8, d) if ard else np.array([0.5])
    m = gp.KernelModel(fam, 1.0, ls, 0.3)
    r = gp.mll_value_and_grad(m, X, y, gp.plan_partitions(n, 64), gp.WorkerPool(),
                              likelihood.CgConfig(tolerance=1.0, probes=10, precond_rank=20), 0)
    assert np.isfinite(r.value)
print("mll ok", flush=True)
cache = predictor.build_cache(gp.KernelModel("matern32", 1.0, np.linspace(0.4, 0.8, d), 0.3), X, y)
Xt = rng.uniform(size=(37, d))
mu = predictor.predict_mean(cache, Xt)
out = predictor.predict(cache, Xt)
assert np.all(np.isfinite(mu)) and np.all(np.isfinite(out.variance))
torch.cuda.synchronize()
print("sanitize workload ok", flush=True)
