"""Run one fused K·V launch (for ncu captures): python scripts/kv_once.py ALGO N D FAM [REPS]."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402

algo, n, d, fam = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
X = syn.whitened_inputs(n, d, 0)
m = gp.KernelModel(fam, 1.0, np.linspace(0.75, 1.5, d), 0.1)
ps = D.points(X)
Xs32, _ = ps.scaled(m.lengthscales)
op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.1, 0, algo=algo, self_offset=0)
V32 = torch.from_numpy(syn.rhs_block(n, 11, 2)).float().cuda()
out = op.apply32(V32, 11)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.apply32(V32, 11, out)
e1.record()
torch.cuda.synchronize()
print(f"algo={algo} n={n} d={d} {fam}: {e0.elapsed_time(e1) / reps:.3f} ms/launch")
