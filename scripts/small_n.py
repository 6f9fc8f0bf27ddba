"""Warm latency of one mll_value_and_grad at small n (C1-shaped by default),
median of REPS calls after 3 warm-up calls, with the stage split of the last
call (run on a B200):  python scripts/small_n.py [workload] [n] [reps]"""

import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as LK, synthetic as syn  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "C1"
    w = syn.WORKLOADS[key]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else w.n
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    kstage = int(sys.argv[4]) if len(sys.argv) > 4 else 10   # repetitions per stage timing
    X = syn.whitened_inputs(n, w.d, 0)
    y = syn.rff_target(X, features=256)
    m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
    cfg = LK.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank)
    plan = gp.plan_partitions(n, max(1, n // 8))
    pool = gp.WorkerPool()
    ts = []
    warm = 3 if reps > 1 else 1
    for r in range(reps + warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = gp.mll_value_and_grad(m, X, y, plan, pool, cfg, 0)
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(time.perf_counter() - t0)
    print(f"{key} n={n} d={w.d} {w.family} rank={w.rank}: mll_value_and_grad median "
          f"{statistics.median(ts) * 1e3:.2f} ms (min {min(ts) * 1e3:.2f}), {res.diagnostics.iterations} "
          f"CG iterations, value {res.value:.6e}")
    # stage split (warm)
    ps = D.points(X)

    def timed(label, fn, k=kstage):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            out = fn()
        torch.cuda.synchronize()
        print(f"  {label:34s} {(time.perf_counter() - t0) / k * 1e3:8.3f} ms")
        return out

    pc = timed("preconditioner (pivchol + factor)", lambda: LK.build_kernel_preconditioner(m, ps, w.rank))
    Z = timed("probes", lambda: LK.draw_probes_device(n, 10, 0, pc))
    op = LK.training_operator(m, ps)
    B = torch.cat([(D.to_device(y) - m.mean)[:, None], Z], 1).contiguous()
    sol = timed("mBCG solve", lambda: LK.mbcg_device(op, B, 1.0, 1000, pc))
    a, S = sol.U[:, 0].contiguous(), sol.U[:, 1:].contiguous()
    timed("SLQ logdet (host)", lambda: LK.slq_logdet(sol, pc, columns=range(1, 11)))
    W = timed("W = P^-1 Z", lambda: LK._pc.precond_apply_device(pc, Z))
    timed("gradient (operands + sym pass)", lambda: LK._gradients(m, ps, a, S, W, pc))


if __name__ == "__main__":
    main()
