"""One wide K·V launch (for ncu): python scripts/wide_once.py N D FAM T"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
n, d, fam, t = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
X = syn.whitened_inputs(n, d, 0)
m = gp.KernelModel(fam, 1.0, np.linspace(0.75, 1.5, d), 0.1)
ps = D.points(X)
Xs32, _ = ps.scaled(m.lengthscales)
op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.1, 0, algo=0)
V32 = torch.from_numpy(np.random.default_rng(1).standard_normal((n, t))).float().cuda()
out = op.apply32(V32, t)
torch.cuda.synchronize()
print("ok")
