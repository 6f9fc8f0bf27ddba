"""Accuracy + timing of the production K·V kernel for one library build:
python scripts/ex2_sweep.py  (uses whatever _lib/libgpbbmm.so is in place)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402

def op_for(n, d, fam, algo):
    X = syn.whitened_inputs(n, d, 0)
    m = gp.KernelModel(fam, 1.0, np.linspace(0.75, 1.5, d), 0.1)
    Xs32, _ = D.points(X).scaled(m.lengthscales)
    return _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.1, 0, algo=algo, self_offset=0)

for fam in ("matern32", "rbf"):
    n, d = 65536, 11
    V = torch.from_numpy(syn.rhs_block(n, 11, 2)).float().cuda()
    a = op_for(n, d, fam, 2).apply32(V, 11).double()
    b = op_for(n, d, fam, 1).apply32(V, 11).double()
    colrel = ((a - b).norm(dim=0) / b.norm(dim=0)).max().item()
    print(f"{fam} n={n}: colrel vs FFMA = {colrel:.3e}, maxabs {((a-b).abs().max()).item():.3e}")
n = 1000000
op = op_for(n, 11, "matern32", 2)
V = torch.from_numpy(syn.rhs_block(n, 11, 2)).float().cuda()
out = op.apply32(V, 11)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    op.apply32(V, 11, out)
e1.record()
torch.cuda.synchronize()
print(f"n=1e6 matern32: {e0.elapsed_time(e1) / 3:.2f} ms/launch")
