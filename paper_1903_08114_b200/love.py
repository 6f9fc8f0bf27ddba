"""LOVE predictive-variance cache (Pleiss et al. 2018, used by the paper for
its one-time prediction precompute).

The reference computes every predictive variance with a batched CG solve
per chunk of test points (predictor.py:135-182), i.e. a fresh n x n solve at
prediction time. LOVE moves that work into a training-data cache: s steps of
block Lanczos on K̂ (block width b, full reorthogonalisation) give
K̂ ≈ Q T Q^T with T block tridiagonal (sb x sb), so K̂^{-1} ≈ R R^T with
R = Q V Λ^{-1/2} (T = V Λ V^T), and

    var(x*) = k(x*, x*) - || R^T k(X, x*) ||^2,

an O(n) cross-kernel product per test point with no solve. The K̂·Q_j
products are the fused tcgen05 operator (t = b = 16: one symmetric-kernel
launch costs the same as t = 1, so a rank-112 cache takes 7 operator
applications); R^T k(X, x*) is the wide cross-kernel product (t = sb <= 256,
csrc/kv_wide.cu). Block orthogonalisation and the small eigenproblem are
plain fp64 BLAS/LAPACK calls on the device.

The cache is an approximation whose error falls with the rank (exact at
sb = n); tests/test_gpu_love.py measures it against the exact CG variances.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _ops
from .kernels import KernelModel
from .likelihood import training_operator


@dataclass
class LoveCache:
    model: KernelModel
    X_train: object
    R: object                      # (n, sb) fp64 on the device: K̂^{-1} ≈ R R^T
    rank: int
    block: int
    steps: int
    ritz: np.ndarray               # eigenvalues of T (Ritz values of K̂), ascending
    diagnostics: dict = field(default_factory=dict)


def _orth(W, Qs):
    """W minus its components in span(Qs), twice (classical Gram-Schmidt with
    reorthogonalisation: the Lanczos basis stays orthogonal to fp64 round-off)."""
    for _ in range(2):
        for Q in Qs:
            W = W - Q @ (Q.T @ W)
    return W


def build_love_cache(model: KernelModel, X, rank: int = 112, block: int = 16, seed: int = 0,
                     precision: str = "fp32") -> LoveCache:
    """Block Lanczos of K̂ = K(X, X) + noise I from a seeded Gaussian block,
    rank = steps x block columns (capped at n)."""
    T = D.torch()
    ps = D.points(X)
    n = ps.n
    model.scale_for(ps.d)
    b = max(1, min(block, n))
    steps = max(1, math.ceil(min(rank, n) / b))
    op = training_operator(model, ps, precision=precision)
    rng = np.random.default_rng(seed)
    Q, _ = T.linalg.qr(D.to_device(rng.standard_normal((n, b))))
    Qs, As, Bs = [Q], [], []
    for j in range(steps):
        W = op(Q)
        A = Q.T @ W
        A = 0.5 * (A + A.T)
        As.append(A)
        if j == steps - 1 or sum(q.shape[1] for q in Qs) >= n:
            break
        W = _orth(W, Qs)
        Qn, Bj = T.linalg.qr(W)
        rem = n - sum(q.shape[1] for q in Qs)
        if rem < Qn.shape[1]:   # the last block of a full-rank basis
            Qn, Bj = Qn[:, :rem], Bj[:rem]
        # a (numerically) rank-deficient block ends the Krylov space
        if float(T.abs(T.diagonal(Bj)).min()) <= 1e-12 * float(T.abs(A).max()):
            break
        Bs.append(Bj)
        Qs.append(Qn)
        Q = Qn
    s = len(As)
    Qs = Qs[:s]
    m = sum(q.shape[1] for q in Qs)
    Tm = T.zeros((m, m), dtype=T.float64, device=D.device())
    off = 0
    for j in range(s):
        bj = Qs[j].shape[1]
        Tm[off:off + bj, off:off + bj] = As[j]
        if j + 1 < s:
            bn = Qs[j + 1].shape[1]
            Tm[off + bj:off + bj + bn, off:off + bj] = Bs[j]
            Tm[off:off + bj, off + bj:off + bj + bn] = Bs[j].T
        off += bj
    lam, V = T.linalg.eigh(Tm)
    # K̂ >= noise I: Ritz values below it are round-off; floor them there
    lam = T.clamp_min(lam, model.noise)
    R = T.cat(Qs, dim=1) @ (V * lam.rsqrt())
    return LoveCache(model=model, X_train=ps, R=R.contiguous(), rank=m, block=b, steps=s,
                     ritz=D.to_host(lam), diagnostics={"precision": precision})


def predict_variance_love_device(cache: LoveCache, X_test, precision: str = "fp32"):
    """k(x*, x*) - ||R^T k(X, x*)||^2 per test point (latent variance, like
    predictor.py's), clamped at 1e-12; returns (variances, clamped count)."""
    T = D.torch()
    model = cache.model
    tr = cache.X_train
    te = D.points(np.atleast_2d(X_test) if not D.is_tensor(X_test) else X_test)
    if te.d != tr.d:
        raise ValueError(f"test points have dimension {te.d}, training data has {tr.d}")
    ls = model.scale_for(tr.d)
    Xr32, Xr64 = te.scaled(ls)
    Xc32, Xc64 = tr.scaled(ls)
    m = cache.R.shape[1]
    if precision == "fp64":
        M, _ = _ops.kv_f64(model.family_code, tr.d, Xr64, Xc64, model.outputscale, 0.0, -1, cache.R)
    elif precision == "fp32":
        # the wide tcgen05 kernel takes up to 256 right-hand sides per pass
        kv = _ops.FusedKernelOperator(model.family_code, tr.d, Xr32, Xc32, model.outputscale, 0.0, -1)
        R32 = cache.R.to(T.float32)
        M = T.cat([kv.apply32(R32[:, c:c + 256].contiguous(), min(256, m - c)).to(T.float64)
                   for c in range(0, m, 256)], dim=1)
    else:
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")
    var = model.outputscale - (M * M).sum(dim=1)
    low = var < 1e-12
    var = T.where(low, T.full_like(var, 1e-12), var)
    return var, int(low.sum().item())


def predict_variance_love(cache: LoveCache, X_test, precision: str = "fp32"):
    var, clamped = predict_variance_love_device(cache, X_test, precision)
    return D.to_host(var), clamped
