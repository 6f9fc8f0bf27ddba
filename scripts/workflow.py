"""End-to-end exact-GP workflow timing on one GPU through the public API
(blockgp-compatible): MLL + gradients, prediction cache, predictive mean and
variance, for a BASELINE.json configuration. Prints one JSON line per stage.

python scripts/workflow.py C2 [--m 1000] [--skip-variance] [--skip-cache] [--train] [--love RANK]
"""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import likelihood, predictor, synthetic as syn  # noqa: E402


def timed(label, fn, **extra):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"stage": label, "seconds": round(dt, 3), **extra}), flush=True)
    return out


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "C2"
    m_test = int(sys.argv[sys.argv.index("--m") + 1]) if "--m" in sys.argv else 1000
    w = syn.WORKLOADS[key]
    X = syn.whitened_inputs(w.n, w.d, 0)
    y = syn.rff_target(X)
    Xt = syn.test_points(m_test, w.d)
    model = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    plan = gp.plan_partitions(w.n, max(1, min(w.n, 2 ** 30 // (8 * w.n))))
    cfg = likelihood.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank)
    gp.mll_value_and_grad(model, X[:4096], y[:4096], gp.plan_partitions(4096, 4096), gp.WorkerPool(), cfg, 0)
    res = timed("mll_value_and_grad", lambda: gp.mll_value_and_grad(model, X, y, plan, gp.WorkerPool(), cfg, 0),
                workload=key, n=w.n, d=w.d)
    print(json.dumps({"stage": "mll_result", "value": res.value, "iterations": res.diagnostics.iterations,
                      "gradients": {k: float(v) for k, v in res.gradients.items()}}), flush=True)
    if "--train" in sys.argv:
        from paper_1903_08114_b200 import trainer as tr
        cfgt = tr.TrainConfig(protocol="pretrain-finetune", family=w.family, ard=w.ard,
                              cg=likelihood.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank))
        mdl, trace = timed("train(pretrain-finetune: 10k-subset L-BFGS 10 + Adam 10, full Adam 3)",
                           lambda: tr.train(X, y, cfgt))
        for r in trace.records:
            print(json.dumps({"stage": "train_step", "phase": r.phase, "step": r.step, "mll": r.mll,
                              "seconds": round(r.seconds, 3), "cg_iterations": r.cg_iterations}), flush=True)
        model = mdl
    if "--skip-cache" in sys.argv:
        return
    cache = timed("build_cache(tol=1e-3)", lambda: predictor.build_cache(model, X, y, precond_rank=w.rank))
    print(json.dumps({"stage": "cache_diag", **{k: (v if not isinstance(v, np.ndarray) else v.tolist())
                                                 for k, v in cache.diagnostics.items()}}, default=str), flush=True)
    mean = timed("predict_mean", lambda: predictor.predict_mean(cache, Xt), m=m_test)
    if "--skip-variance" in sys.argv:
        return
    var, clamped = timed("predict_variance(tol=0.01)",
                         lambda: predictor.predict_variance(cache, Xt, precond_rank=w.rank), m=m_test)
    print(json.dumps({"stage": "pred_summary", "mean_abs": float(np.abs(mean).mean()),
                      "var_min": float(var.min()), "var_max": float(var.max()), "clamped": clamped}), flush=True)
    if "--love" in sys.argv:
        from paper_1903_08114_b200 import love
        rank = int(sys.argv[sys.argv.index("--love") + 1])
        lc = timed(f"build_love_cache(rank={rank})", lambda: love.build_love_cache(model, X, rank=rank))
        lv, _ = timed("predict_variance_love", lambda: love.predict_variance_love(lc, Xt), m=m_test)
        print(json.dumps({"stage": "love_vs_cg", "max_abs_diff": float(np.abs(lv - var).max()),
                          "median_abs_diff": float(np.median(np.abs(lv - var))),
                          "mean_var": float(var.mean())}), flush=True)


if __name__ == "__main__":
    main()
