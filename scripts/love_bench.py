"""LOVE cache vs the reference-semantics CG variances (predictor.py:135-182):
build / predict time and accuracy (GPU).  python scripts/love_bench.py WORKLOAD [n_test] [ranks...]"""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import love, predictor, synthetic as syn  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


key = sys.argv[1] if len(sys.argv) > 1 else "C2"
n_test = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ranks = [int(r) for r in sys.argv[3:]] or [112, 256]
w = syn.WORKLOADS[key]
X = syn.whitened_inputs(w.n, w.d, 0)
Xt = syn.whitened_inputs(n_test, w.d, 7) * 1.05
m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
cache = predictor.PredictionCache(model=m, X_train=X, weights=np.zeros(w.n), cache_tolerance=0.01)
(ref01, _), t_cg = timed(lambda: predictor.predict_variance(cache, Xt, precond_rank=w.rank))
# the accuracy reference: the same CG variances at a tight tolerance
(ref, clamped), t_tight = timed(lambda: predictor.predict_variance(cache, Xt, precond_rank=w.rank, tolerance=1e-6))
out = {"workload": key, "n": w.n, "n_test": n_test, "cg_variance_s": t_cg, "cg_tolerance": 0.01,
       "cg_tol001_max_abs_err": float(np.abs(ref01 - ref).max()), "cg_tight_s": t_tight, "love": []}
for r in ranks:
    lc, t_build = timed(lambda: love.build_love_cache(m, X, rank=r, block=16))
    (v, _), t_pred = timed(lambda: love.predict_variance_love(lc, Xt))
    err = np.abs(v - ref)
    out["love"].append({"rank": lc.rank, "build_s": t_build, "predict_s": t_pred,
                        "max_abs_err": float(err.max()), "median_abs_err": float(np.median(err)),
                        "max_rel_err": float((err / ref).max()), "mean_var": float(ref.mean())})
print(json.dumps(out))
