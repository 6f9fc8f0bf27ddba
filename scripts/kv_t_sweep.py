"""K·V launch time vs right-hand-side count t at a workload's n and d
(row-tiled / default dispatch): python scripts/kv_t_sweep.py C4 [algo] (B200)."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = syn.WORKLOADS[key]
X = syn.whitened_inputs(w.n, w.d, 0)
m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
ps = D.points(X)
Xs32, _ = ps.scaled(m.scale_for(w.d))
op = _ops.FusedKernelOperator(m.family_code, w.d, Xs32, Xs32, 1.0, 0.0, -1, algo=algo, self_offset=0)
for t in (1, 4, 11, 16, 32, 64, 128, 256):
    V = torch.randn(w.n, t, device="cuda")
    out = op.apply32(V, t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.apply32(V, t, out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{key} n={w.n} d={w.d} t={t:3d} algo={algo}: {e0.elapsed_time(e1):9.2f} ms", flush=True)
