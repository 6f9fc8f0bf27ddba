"""C2 gradients (fp64 operator, eps = 1): fused forms (tcgen05 ARD and SIMT)
against a dense fp64 evaluation of the reference's formula
(likelihood.py:166-216) on the SAME solves a, S, W — separates the gradient
pass's own error from solve differences. Diagnostic only (GPU)."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))

import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, likelihood as L, synthetic as syn  # noqa: E402
from conftest import load_golden  # noqa: E402

SQRT3 = 3.0 ** 0.5


def dense_grads(model, ps, a, S, W, cache):
    T = D.torch()
    n, t = W.shape
    ls = model.scale_for(ps.d)
    _, X64 = ps.scaled(ls)
    R = T.cat([a[:, None], W] + ([cache.factor_device] if cache is not None else []), dim=1)
    d = ps.d
    GR = [T.zeros_like(R) for _ in range(1 + d)]
    blk = 2048
    for s in range(0, n, blk):
        e = min(n, s + blk)
        A = X64[s:e]
        Dsq = T.cdist(A, X64).square_()
        r = Dsq.sqrt()
        if model.family == "rbf":
            K = model.outputscale * T.exp(-0.5 * Dsq)
            env = K
        else:
            K = model.outputscale * (1 + SQRT3 * r) * T.exp(-SQRT3 * r)
            env = 3.0 * model.outputscale * T.exp(-SQRT3 * r)
        GR[0][s:e] = (K / model.outputscale) @ R
        for i in range(d):
            diff = (A[:, i, None] - X64[None, :, i]) ** 2
            GR[1 + i][s:e] = (env * diff / float(ls[i])) @ R
    out = {}
    names = ["outputscale"] + [f"lengthscale_{i}" for i in range(d)]
    Lf = cache.factor_device
    B = cache.noise * T.eye(Lf.shape[1], dtype=T.float64, device=Lf.device) + Lf.T @ Lf
    for p, G in zip(names, GR):
        quad = float(a @ G[:, 0])
        trG = n if p == "outputscale" else 0.0
        inner = T.linalg.solve(B, Lf.T @ G[:, 1 + t:])
        exact = (trG - float(T.trace(inner))) / cache.noise
        resid = float(((S - W) * G[:, 1:1 + t]).sum()) / t
        out[p] = (0.5 * quad - 0.5 * (exact + resid), quad, exact, resid)
    return out


def main():
    g = load_golden("c2_mll")
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(w.n, w.d, 0)
    y = syn.rff_target(X, seed=1)
    m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    cap = {}
    orig = L._gradients

    def spy(model, ps, a, S, W, cache):
        cap.update(model=model, ps=ps, a=a, S=S, W=W, cache=cache)
        return orig(model, ps, a, S, W, cache)

    L._gradients = spy
    prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
    res = gp.mll_value_and_grad(m, X, y, gp.plan_from_budget(w.n), gp.WorkerPool(),
                                L.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank, precision=prec), 0)
    print("iterations", res.diagnostics.iterations, "ref", int(g["iterations"]))
    keys = [str(k) for k in g["grad_keys"]]
    ref = dict(zip(keys, g["grad_vals"]))
    md, ps = cap["model"], cap["ps"]
    dn = dense_grads(md, ps, cap["a"], cap["S"], cap["W"], cap["cache"])
    Y, R = L.gradient_operands(cap["a"], cap["S"], cap["W"], cap["cache"])
    Xs32 = ps.scaled(md.scale_for(ps.d))[0]
    simt_raw = L._grad_forms_raw(md, ps.d, Xs32, Xs32, Y, R, algo=1)
    simt = L.assemble_gradients(md, simt_raw, cap["a"], cap["S"], cap["W"], cap["cache"], w.n)
    T = D.torch()
    for algo in (1, 2, 3):
        L._grad_forms_raw(md, ps.d, Xs32, Xs32, Y, R, algo=algo)
        T.cuda.synchronize()
        e0, e1 = T.cuda.Event(enable_timing=True), T.cuda.Event(enable_timing=True)
        e0.record()
        raw = L._grad_forms_raw(md, ps.d, Xs32, Xs32, Y, R, algo=algo)
        e1.record()
        T.cuda.synchronize()
        gg = L.assemble_gradients(md, raw, cap["a"], cap["S"], cap["W"], cap["cache"], w.n)
        err = max(abs(gg[k] - dn[k][0]) for k in dn) / np.abs(g["grad_vals"]).max()
        print(f"algo {algo}: {e0.elapsed_time(e1):.2f} ms, max |g - dense64| / max|g| = {err:.2e}")
    Ys, Rs = L.symmetric_gradient_operands(cap["a"], cap["S"], cap["W"], cap["cache"])
    L._grad_forms_sym_raw(md, ps.d, Xs32, Ys, Rs)
    T.cuda.synchronize()
    e0, e1 = T.cuda.Event(enable_timing=True), T.cuda.Event(enable_timing=True)
    e0.record()
    raw = L._grad_forms_sym_raw(md, ps.d, Xs32, Ys, Rs)
    e1.record()
    T.cuda.synchronize()
    gg = L.assemble_gradients(md, raw, cap["a"], cap["S"], cap["W"], cap["cache"], w.n)
    err = max(abs(gg[k] - dn[k][0]) for k in dn) / np.abs(g["grad_vals"]).max()
    print(f"symmetric grad_tc: {e0.elapsed_time(e1):.2f} ms, max |g - dense64| / max|g| = {err:.2e}")
    mx = np.abs(g["grad_vals"]).max()
    print(f"{'param':>14} {'reference':>12} {'fused':>12} {'simt':>12} {'dense64':>12}  quad exact resid")
    for k in keys:
        if k in dn:
            v = dn[k]
            print(f"{k:>14} {ref[k]:12.3f} {res.gradients[k]:12.3f} {simt[k]:12.3f} {v[0]:12.3f}  "
                  f"{v[1]:.4e} {v[2]:.4e} {v[3]:.4e}")
        else:
            print(f"{k:>14} {ref[k]:12.3f} {res.gradients[k]:12.3f} {simt.get(k, float('nan')):12.3f}")
    print("max |fused - ref| / max", max(abs(res.gradients[k] - ref[k]) for k in keys) / mx)
    print("max |dense64 - ref| / max", max(abs(dn[k][0] - ref[k]) for k in dn) / mx)


if __name__ == "__main__":
    main()
