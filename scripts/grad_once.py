"""One fused gradient pass (for ncu / timing): python scripts/grad_once.py N D FAM ARD W"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as LK, synthetic as syn  # noqa: E402
n, d, fam, ard, w = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
X = syn.whitened_inputs(n, d, 0)
ls = np.linspace(0.75, 1.5, d) if ard else np.array([1.0])
m = gp.KernelModel(fam, 1.0, ls, 0.1)
ps = D.points(X)
Xs32, _ = ps.scaled(m.scale_for(d))
rng = np.random.default_rng(0)
Y = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
R = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
out = LK._grad_forms_raw(m, d, Xs32, Xs32, Y, R)
torch.cuda.synchronize()
t0 = time.perf_counter()
out = LK._grad_forms_raw(m, d, Xs32, Xs32, Y, R)
torch.cuda.synchronize()
print(f"grad n={n} d={d} {fam} ard={ard} w={w}: {(time.perf_counter() - t0) * 1e3:.1f} ms")
