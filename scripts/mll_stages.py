"""Stage timing of one mll_value_and_grad at a given workload (run on a B200).

    python scripts/mll_stages.py [workload] [n]
"""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as LK, synthetic as syn  # noqa: E402
from paper_1903_08114_b200 import precond as PC  # noqa: E402
from paper_1903_08114_b200.cg import MbcgRun  # noqa: E402


def timed(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{label:38s} {dt * 1e3:10.1f} ms", flush=True)
    return out, dt


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "M1e6"
    w = syn.WORKLOADS[key]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else w.n
    X = syn.whitened_inputs(n, w.d, 0)
    y = syn.rff_target(X, features=256)
    m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
    ps = D.points(X)
    ps.scaled(m.lengthscales)
    print(f"{key}: n={n} d={w.d} {w.family} ard={w.ard} rank={w.rank}")
    pc, _ = timed("pivoted Cholesky + factor", lambda: LK.build_kernel_preconditioner(m, ps, w.rank))
    Z, _ = timed("probes", lambda: LK.draw_probes_device(n, 10, 0, pc))
    op = LK.training_operator(m, ps)
    B = torch.cat([D.to_device(y)[:, None], Z], 1)
    run, _ = timed("mBCG init", lambda: MbcgRun(op, B, 1.0, 1000, pc))
    t0 = time.perf_counter()
    while run.step():
        pass
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{'mBCG (tol 1) ' + str(run.iterations) + ' iterations':38s} {dt * 1e3:10.1f} ms "
          f"({dt / run.iterations * 1e3:.1f} ms/iter)")
    sol = run.finish()
    a, S = sol.U[:, 0].contiguous(), sol.U[:, 1:].contiguous()
    W, _ = timed("W = P^-1 Z", lambda: PC.precond_apply_device(pc, Z))
    YR, _ = timed("gradient operands", lambda: LK.gradient_operands(a, S, W, pc))
    Xs32, _ = ps.scaled(m.lengthscales)
    raw, _ = timed("fused gradient pass", lambda: LK._grad_forms_raw(m, ps.d, Xs32, Xs32, *YR))
    t0 = time.perf_counter()
    res = gp.mll_value_and_grad(m, X, y, gp.plan_partitions(n, max(1, n // 8)), gp.WorkerPool(),
                                LK.CgConfig(), 0)
    print(f"{'full mll_value_and_grad':38s} {(time.perf_counter() - t0) * 1e3:10.1f} ms  "
          f"value={res.value:.6e} iters={res.diagnostics.iterations}")


if __name__ == "__main__":
    main()
