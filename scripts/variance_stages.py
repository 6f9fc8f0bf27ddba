"""Cost split of one predictive-variance chunk (256 test points) at a workload
(run on a B200): python scripts/variance_stages.py [C2]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as LK, synthetic as syn  # noqa: E402
from paper_1903_08114_b200.cg import MbcgRun  # noqa: E402
from paper_1903_08114_b200.predictor import kernel_block_device  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = syn.WORKLOADS[key]
X = syn.whitened_inputs(w.n, w.d, 0)
m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
Xt = syn.whitened_inputs(256, w.d, 3)
ps = D.points(X)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pc = LK.build_kernel_preconditioner(m, ps, 100)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    Bm = kernel_block_device(m, ps, Xt).contiguous()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    op = LK.training_operator(m, ps)
    run = MbcgRun(op, Bm, 0.01, 1000, pc)
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    run.kv_events = ev
    kv = 0.0
    while True:
        act = run.step()
        kv += ev[0].elapsed_time(ev[1])
        if act == 0:
            break
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"{key} n={w.n} chunk 256: precond {1e3*(t1-t0):.1f} ms, B block {1e3*(t2-t1):.1f} ms, "
          f"mBCG {run.iterations} iterations {1e3*(t3-t2):.1f} ms (K·V {kv:.1f} ms, "
          f"{kv/run.iterations:.2f} ms/iter)", flush=True)
