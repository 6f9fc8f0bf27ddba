"""cProfile of warm mll_value_and_grad calls at small n (host-side overhead
between kernels): python scripts/host_profile.py [workload] [reps] (B200)."""

import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import likelihood as LK, synthetic as syn  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
w = syn.WORKLOADS[key]
X = syn.whitened_inputs(w.n, w.d, 0)
y = syn.rff_target(X, features=256)
m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
cfg = LK.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank)
plan = gp.plan_partitions(w.n, max(1, w.n // 8))
for _ in range(3):
    gp.mll_value_and_grad(m, X, y, plan, gp.WorkerPool(), cfg, 0)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    gp.mll_value_and_grad(m, X, y, plan, gp.WorkerPool(), cfg, 0)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
st.sort_stats("cumulative").print_stats("paper_1903_08114_b200", 60)
