"""C2 (eps = 1) solve in both operator precisions against the reference's
per-iteration recurrence residuals (tests/golden/c2_mll.npz): where the
trajectories part (diagnostic, GPU)."""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))

import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as L, synthetic as syn  # noqa: E402
from conftest import load_golden  # noqa: E402

g = load_golden("c2_mll")
w = syn.WORKLOADS["C2"]
X = syn.whitened_inputs(w.n, w.d, 0)
y = syn.rff_target(X, seed=1)
m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
ps = D.points(X)
pc = L.build_kernel_preconditioner(m, ps, w.rank)
Z = L.draw_probes_device(w.n, 10, 0, pc)
Zh = D.to_host(Z)
print("Z checksum", [Zh.sum(), (Zh * Zh).sum()], "ref", g["Z_checksum"])
B = torch.cat([(D.to_device(y) - m.mean)[:, None], Z], 1).contiguous()
H = g["residual_history"]
for prec in ("fp64", "fp32"):
    op = L.training_operator(m, ps, precision=prec)
    sol = L.mbcg_device(op, B, 1.0, 1000, pc)
    R = sol.residual_history if hasattr(sol, "residual_history") else sol.history
    its = min(R.shape[0], H.shape[0])
    d = np.abs(R[:its] - H[:its]) / np.abs(H[:its])
    print(prec, "iterations", sol.iterations, "ref", H.shape[0])
    np.set_printoptions(linewidth=200, precision=1)
    for i in range(its):
        print(f"  it {i + 1:3d} max rel diff {d[i].max():.2e}  per column " + " ".join(f"{x:.0e}" for x in d[i]))
    if prec == "fp64":
        # our own sensitivity: y[0] moved by one ulp (the reference moves by 1e-15, c2_ulp golden)
        y2 = y.copy()
        y2[0] = np.nextafter(y2[0], np.inf)
        B2 = torch.cat([(D.to_device(y2) - m.mean)[:, None], Z], 1).contiguous()
        sol2 = L.mbcg_device(op, B2, 1.0, 1000, pc)
        R2 = sol2.history
        d2 = np.abs(R2[:its] - R[:its]) / np.abs(R[:its])
        print("  fp64, y + 1 ulp vs fp64: per-iteration max rel diff", " ".join(f"{x:.0e}" for x in d2.max(axis=1)))
