"""torch.profiler trace of one warm mll_value_and_grad (C1 by default):
kernel list with durations and the host gaps between them (run on a B200)."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import likelihood as LK, synthetic as syn  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
w = syn.WORKLOADS[key]
X = syn.whitened_inputs(w.n, w.d, 0)
y = syn.rff_target(X, features=256)
m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
cfg = LK.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank)
plan = gp.plan_partitions(w.n, max(1, w.n // 8))
for _ in range(3):
    gp.mll_value_and_grad(m, X, y, plan, gp.WorkerPool(), cfg, 0)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    gp.mll_value_and_grad(m, X, y, plan, gp.WorkerPool(), cfg, 0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
tot = 0.0
prev_end = t0
print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>8}  kernel")
for e in evs:
    gap = e.time_range.start - prev_end
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.elapsed_us():8.1f} {gap:8.1f}  {e.name[:90]}")
    tot += e.time_range.elapsed_us()
    prev_end = e.time_range.end
print(f"kernels: {len(evs)}, busy {tot:.1f} us, span {prev_end - t0:.1f} us")
