"""Per-iteration cost split of the mBCG solver at a workload (run on a B200):
K·V kernel time (CUDA events) vs the whole step (host loop included).
    python scripts/step_overhead.py C2
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as LK, synthetic as syn  # noqa: E402
from paper_1903_08114_b200.cg import MbcgRun  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = syn.WORKLOADS[key]
X = syn.whitened_inputs(w.n, w.d, 0)
y = syn.rff_target(X)
m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
ps = D.points(X)
pc = LK.build_kernel_preconditioner(m, ps, w.rank)
Z = LK.draw_probes_device(w.n, 10, 0, pc)
op = LK.training_operator(m, ps)
B = torch.cat([D.to_device(y)[:, None], Z], 1)
for rep in range(2):
    run = MbcgRun(op, B, 1e-300, 30, pc)
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    run.kv_events = ev
    kv = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        run.step()
        kv.append(ev[0].elapsed_time(ev[1]))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20 * 1e3
print(f"{key}: step {dt:.3f} ms, K·V {sum(kv) / len(kv):.3f} ms, rest {dt - sum(kv) / len(kv):.3f} ms")
