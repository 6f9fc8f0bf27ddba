"""Time the CG Woodbury phases at the bench's shape (n = 10^6, t = 11,
k = 100): gp_mbcg_update (alpha/U/R update + L^T R) and gp_mbcg_precond
(Z = P^{-1} R), REPS launches each after one real mBCG step, CUDA events on
the library's stream. python scripts/woodbury_once.py [n] [reps]"""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
from paper_1903_08114_b200.cg import FusedOperator, MbcgRun  # noqa: E402
from paper_1903_08114_b200.likelihood import build_kernel_preconditioner, draw_probes_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = syn.WORKLOADS["M1e6"]
X = syn.whitened_inputs(n, w.d, 0)
y = syn.rff_target(X, features=256)
model = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
ps = D.points(X)
Xs32, _ = ps.scaled(model.lengthscales)
pc = build_kernel_preconditioner(model, ps, w.rank)
Z = draw_probes_device(n, 10, 0, pc)
B = torch.cat([D.to_device(y)[:, None], Z], dim=1).contiguous()
kv = _ops.training_operator(model.family_code, w.d, Xs32, 1.0, 0.0, -1)
run = MbcgRun(FusedOperator(kv, model.noise, n), B, 1e-300, 5, pc)
run.step()
torch.cuda.synchronize()
ph = run.ph


def timed(label, fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call")


timed("precond (Z = P^-1 R)", lambda: ph.precond(1, 1e-300))
timed("update (U, R, L^T R)", lambda: ph.update(run.Q, run.f64, 1))
