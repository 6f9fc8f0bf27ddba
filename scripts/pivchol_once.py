"""Time the pivoted-Cholesky factor (gp_pivchol) at the bench shape:
python scripts/pivchol_once.py [n] [k] [reps]"""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, precond, synthetic as syn  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
w = syn.WORKLOADS["M1e6"]
X = syn.whitened_inputs(n, w.d, 0)
m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
src = precond.KernelRowSource(m, X)
f = precond.partial_pivoted_cholesky(src, np.full(n, 1.0), k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    f = precond.partial_pivoted_cholesky(src, np.full(n, 1.0), k)
torch.cuda.synchronize()
print(f"pivchol n={n} k={k}: {(time.perf_counter() - t0) / reps * 1e3:.2f} ms, pivots[:5]={list(f.pivots[:5])}")
