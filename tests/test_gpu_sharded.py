"""Row-sharded MLL + gradients and predictive mean with two
ranks sharing one GPU over gloo: the multi-GPU code path (all-gather of the
search directions and of a, all-reduce of the CG payload and of the
gradient partial sums) against the single-process result."""

import os
import tempfile

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _rank_main(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1903_08114_b200 as gp
    from paper_1903_08114_b200 import likelihood, sharded
    from paper_1903_08114_b200.distributed import TorchComm
    g = load_golden("c1_full")
    X, y = g["X"], g["y"]
    model = gp.KernelModel("matern32", 1.0, np.linspace(0.75, 1.5, 8) * 0.5, 0.2)
    comm = TorchComm(X.shape[0])
    cfg = likelihood.CgConfig(tolerance=0.01, probes=10, precond_rank=50)
    res = sharded.mll_value_and_grad_sharded(model, X, y, cfg, 3, comm)
    w = np.random.default_rng(1).standard_normal(X.shape[0])
    Xt = np.random.default_rng(2).uniform(size=(300, 8))
    mean = sharded.predict_mean_sharded(model, X, w, Xt, comm)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), value=res.value, iters=res.diagnostics.iterations,
             keys=np.array(list(res.gradients)), grads=np.array(list(res.gradients.values())), mean=mean)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_mll_and_mean_match_single_process():
    import torch.multiprocessing as mp
    import paper_1903_08114_b200 as gp
    from paper_1903_08114_b200 import likelihood, predictor
    g = load_golden("c1_full")
    X, y = g["X"], g["y"]
    model = gp.KernelModel("matern32", 1.0, np.linspace(0.75, 1.5, 8) * 0.5, 0.2)
    cfg = likelihood.CgConfig(tolerance=0.01, probes=10, precond_rank=50)
    # the shards run the row-tiled kernel; compare against the same kernel on
    # the whole operator (the single-GPU default is the symmetric kernel,
    # equal to it only within fp32 round-off)
    os.environ["GP_KV_NO_SYM"] = "1"
    try:
        ref = gp.mll_value_and_grad(model, X, y, gp.plan_partitions(4096, 4096), gp.WorkerPool(), cfg, 3)
    finally:
        del os.environ["GP_KV_NO_SYM"]
    sym = gp.mll_value_and_grad(model, X, y, gp.plan_partitions(4096, 4096), gp.WorkerPool(), cfg, 3)
    assert abs(sym.value - ref.value) <= 1e-5 * abs(ref.value)
    w = np.random.default_rng(1).standard_normal(X.shape[0])
    Xt = np.random.default_rng(2).uniform(size=(300, 8))
    cache = predictor.PredictionCache(model=model, X_train=X, weights=w, cache_tolerance=1e-3)
    ref_mean = predictor.predict_mean(cache, Xt)
    with tempfile.TemporaryDirectory() as d:
        port = 29500 + os.getpid() % 1000
        mp.spawn(_rank_main, args=(2, port, d), nprocs=2, join=True)
        outs = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(2)]
    for o in outs:
        assert int(o["iters"]) == ref.diagnostics.iterations
        assert abs(float(o["value"]) - ref.value) <= 1e-7 * abs(ref.value)
        scale = max(abs(v) for v in ref.gradients.values())
        got = dict(zip([str(k) for k in o["keys"]], o["grads"]))
        for k, v in ref.gradients.items():
            assert abs(got[k] - v) <= 1e-6 * scale, (k, got[k], v)
        assert np.linalg.norm(o["mean"] - ref_mean) <= 1e-5 * np.linalg.norm(ref_mean - model.mean)
