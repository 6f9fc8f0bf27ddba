"""C2 stability study (GPU, ~40 GB): the reference's PCG restated in torch
fp64 on the DENSE kernel matrix, with the Woodbury preconditioner applied
(a) via the inner Cholesky (cho_solve, as precond.py:125-139) and (b) via the
explicit inverse B^-1 (as the device mBCG does), against the reference's
residual history and against one another, plus each one's sensitivity to a
1-ulp change of y[0]."""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))

import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, kernels, likelihood as L, synthetic as syn  # noqa: E402
from conftest import load_golden  # noqa: E402

g = load_golden("c2_mll")
w = syn.WORKLOADS["C2"]
X = syn.whitened_inputs(w.n, w.d, 0)
y = syn.rff_target(X, seed=1)
m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
ps = D.points(X)
pc = L.build_kernel_preconditioner(m, ps, w.rank)
Z = L.draw_probes_device(w.n, 10, 0, pc)
K = kernels.kernel_block_device(m, X, X, add_noise=True)   # dense fp64, n x n
Lf = pc.factor_device
noise = pc.noise
Bm = noise * torch.eye(Lf.shape[1], dtype=torch.float64, device=Lf.device) + Lf.T @ Lf
C = torch.linalg.cholesky(Bm)
Binv = pc.binv_device
print("noise", noise, "cond(B)", float(torch.linalg.cond(Bm)))


def papply(R, mode):
    LtR = Lf.T @ R
    c = torch.cholesky_solve(LtR, C) if mode == "chol" else Binv @ LtR
    return (R - Lf @ c) / noise


def pcg(B, mode, tol=1.0, maxit=1000):
    n, t = B.shape
    norms = B.norm(dim=0)
    U = torch.zeros_like(B)
    R = B.clone()
    Zc = papply(R, mode)
    P = Zc.clone()
    gamma = (R * Zc).sum(0)
    active = torch.ones(t, dtype=torch.bool, device=B.device)
    hist = []
    for it in range(1, maxit + 1):
        cols = torch.nonzero(active).flatten()
        V = K @ P[:, cols]
        pv = (P[:, cols] * V).sum(0)
        alpha = gamma[cols] / pv
        U[:, cols] += alpha * P[:, cols]
        R[:, cols] -= alpha * V
        rel = hist[-1].clone() if hist else torch.ones(t, dtype=torch.float64, device=B.device)
        rel[cols] = R[:, cols].norm(dim=0) / norms[cols]
        hist.append(rel)
        done = rel[cols] <= tol
        active[cols[done]] = False
        if not active.any():
            break
        keep = torch.nonzero(active).flatten()
        Zk = papply(R[:, keep], mode)
        gn = (R[:, keep] * Zk).sum(0)
        P[:, keep] = Zk + (gn / gamma[keep]) * P[:, keep]
        gamma[keep] = gn
    return torch.stack(hist).cpu().numpy(), U


H = g["residual_history"]
Bb = torch.cat([(D.to_device(y) - m.mean)[:, None], Z], 1).contiguous()
y2 = y.copy()
y2[0] = np.nextafter(y2[0], np.inf)
Bb2 = torch.cat([(D.to_device(y2) - m.mean)[:, None], Z], 1).contiguous()
sys.path.insert(0, HERE)
from c2_grad_check import dense_grads  # noqa: E402
keys = [str(k) for k in g["grad_keys"]]
ref = dict(zip(keys, g["grad_vals"]))
mx = np.abs(g["grad_vals"]).max()
for mode in ("chol", "inv"):
    h, U = pcg(Bb, mode)
    h2, _ = pcg(Bb2, mode)
    # gradients of the reference formula (likelihood.py:166-216) on these solves
    a, S = U[:, 0].contiguous(), U[:, 1:].contiguous()
    W = papply(Z, "chol")
    dn = dense_grads(m, ps, a, S, W, pc)
    t = Z.shape[1]
    tr_noise = (w.n - (pc.rank - noise * pc.tr_binv)) / noise
    gnoise = 0.5 * float(a @ a) - 0.5 * (tr_noise + float(((S - W) * W).sum()) / t)
    errs = {k: abs(dn[k][0] - ref[k]) / mx for k in dn}
    errs["noise"] = abs(gnoise - ref["noise"]) / mx
    print(f"{mode}: gradient |dense-PCG - reference| / max|g|: " + " ".join(f"{k}={v:.1e}" for k, v in errs.items()))
    its = min(len(h), len(H))
    dref = (np.abs(h[:its] - H[:its]) / np.abs(H[:its])).max(1)
    its2 = min(len(h), len(h2))
    dulp = (np.abs(h[:its2] - h2[:its2]) / np.abs(h[:its2])).max(1)
    print(f"{mode}: iterations {len(h)} (reference {len(H)})")
    print("  vs reference, per iteration:", " ".join(f"{x:.0e}" for x in dref))
    print("  y + 1 ulp, per iteration:   ", " ".join(f"{x:.0e}" for x in dulp))
