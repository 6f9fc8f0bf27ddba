"""Rank-k pivoted-Cholesky preconditioner (mirror of blockgp.precond).

P = L L^T + noise I with L (n x k) from greedy pivoted Cholesky of the
noiseless kernel (precond.py:58-98); applied through Woodbury
(precond.py:125-139). Factor, inner Cholesky and B^{-1} live in HBM; the
kernel-row factorisation runs entirely on the device (gp_pivchol) and the
Woodbury products run through gp_lt_mul / gp_lowrank_mul.
"""

from __future__ import annotations

import math

import numpy as np

from . import _device as D
from . import _lib
from . import _ops
from .errors import NumericError


class PivotedFactor:
    """Rank-k factor from greedy diagonal pivoting (precond.py:19-33).
    `factor`, `pivots`, `residual_diag` are numpy views fetched lazily from
    the device copies (`factor_device`, ...)."""

    def __init__(self, factor_device, pivots, residual_device):
        self.factor_device = factor_device
        self._pivots = np.asarray(pivots, dtype=np.intp)
        self.residual_device = residual_device

    @property
    def factor(self) -> np.ndarray:
        return D.to_host(self.factor_device)

    @property
    def pivots(self) -> np.ndarray:
        return self._pivots

    @property
    def residual_diag(self) -> np.ndarray:
        return D.to_host(self.residual_device)

    @property
    def rank(self) -> int:
        return int(self.factor_device.shape[1])


class PreconditionerCache:
    """Device-resident Woodbury cache for P = L L^T + noise I
    (precond.py:36-55): factor L, lower inner Cholesky of noise I + L^T L,
    its inverse product B^{-1}, logdet P and tr(B^{-1})."""

    def __init__(self, factor_device, noise, chol_device, binv_device, logdet, tr_binv):
        self.factor_device = factor_device
        self.noise = float(noise)
        self.chol_device = chol_device
        self.binv_device = binv_device
        self.logdet = float(logdet)
        self.tr_binv = float(tr_binv)

    @property
    def factor(self) -> np.ndarray:
        return D.to_host(self.factor_device)

    @property
    def inner_chol(self) -> np.ndarray:
        return D.to_host(self.chol_device) if self.rank else np.zeros((0, 0))

    @property
    def n(self) -> int:
        return int(self.factor_device.shape[0])

    @property
    def rank(self) -> int:
        return int(self.factor_device.shape[1])


class KernelRowSource:
    """Row oracle of the noiseless kernel over X (likelihood.py:86-87), in a
    form gp_pivchol consumes directly on the device."""

    def __init__(self, model, X):
        self.model = model
        self.points = D.points(X)

    def __call__(self, i):  # reference-style use: one materialised row
        from .kernels import kernel_rows
        return kernel_rows(self.model, self.points.X, i, i + 1, noise=False)[0]


def _pivchol_device(src: KernelRowSource, k: int, overlap=None):
    T = D.torch()
    ps, model = src.points, src.model
    n = ps.n
    _, Xs64 = ps.scaled(model.scale_for(ps.d))
    L = T.empty((n, k), dtype=T.float64, device=D.device())
    piv = T.empty(k, dtype=T.int64, device=D.device())
    resid = T.empty(n, dtype=T.float64, device=D.device())
    info = T.zeros(1, dtype=T.int32, device=D.device())
    lib = _lib.lib()
    nbytes = lib.gp_pivchol_workspace_bytes(n, k)
    ws = _ops.workspace().bytes("pivchol", nbytes)
    _lib.check(lib.gp_pivchol(model.family_code, ps.d, _lib.ptr(Xs64), ps.d, n,
                              float(model.outputscale), k, _lib.ptr(L), k, _lib.ptr(piv),
                              _lib.ptr(resid), _lib.ptr(info), _lib.ptr(ws), nbytes,
                              _lib.stream_handle()), "gp_pivchol")
    if overlap is not None:   # host work while the factorisation runs
        overlap()
    host = D.to_host(T.cat([piv, info.to(T.int64)]))   # pivots and rank in one read
    rank = int(host[k])
    return PivotedFactor(L[:, :rank], host[:rank].copy(), resid)


def partial_pivoted_cholesky(row_fn, diag, k: int, overlap=None) -> PivotedFactor:
    """Greedy rank-k pivoted Cholesky (precond.py:58-98). Kernel row sources
    run fully on the device; arbitrary row callables are evaluated per pivot
    and the factor updates run on the device."""
    if isinstance(row_fn, KernelRowSource):
        n = row_fn.points.n
        if not 1 <= k <= n:
            raise ValueError(f"rank must satisfy 1 <= k <= {n}, got {k}")
        dg = np.asarray(diag, dtype=np.float64)
        if dg.shape != (n,) or not np.all(dg == row_fn.model.outputscale):
            raise ValueError("kernel row source expects the constant diagonal outputscale")
        return _pivchol_device(row_fn, k, overlap)
    T = D.torch()
    d = D.to_device(diag).clone()
    n = d.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"rank must satisfy 1 <= k <= {n}, got {k}")
    L = T.zeros((n, k), dtype=T.float64, device=D.device())
    piv = []
    for j in range(k):
        i = int(T.argmax(d).item())  # first maximal index, as np.argmax
        di = float(d[i].item())
        if di <= 0.0:
            return PivotedFactor(L[:, :j].clone(), piv, T.clamp_min(d, 0.0))
        piv.append(i)
        row = D.to_device(row_fn(i))
        if tuple(row.shape) != (n,):
            raise ValueError(f"row oracle returned shape {tuple(row.shape)}, expected ({n},)")
        col = (row - L[:, :j] @ L[i, :j]) / math.sqrt(di)
        L[:, j] = col
        d -= col * col
        d.clamp_(min=0.0)
        d[i] = 0.0
    return PivotedFactor(L, piv, d)


def build_preconditioner(factor, noise: float) -> PreconditionerCache:
    """Inner Cholesky of noise I + L^T L, logdet P = (n-k) log noise +
    2 sum log diag, B^{-1} and tr(B^{-1}) (precond.py:101-122, :165-174)."""
    if noise <= 0:
        raise ValueError(f"noise must be positive, got {noise}")
    T = D.torch()
    L = factor.factor_device if isinstance(factor, PivotedFactor) else D.to_device(factor)
    if L.dim() != 2:
        raise ValueError("factor must be an (n, k) matrix")
    L = L.contiguous()
    n, k = L.shape
    if k == 0:
        z = T.zeros((0, 0), dtype=T.float64, device=D.device())
        return PreconditionerCache(L, noise, z, z, n * math.log(noise), 0.0)
    chol = T.empty((k, k), dtype=T.float64, device=D.device())
    binv = T.empty((k, k), dtype=T.float64, device=D.device())
    out = T.zeros(2, dtype=T.float64, device=D.device())
    info = T.zeros(1, dtype=T.int32, device=D.device())
    part = _ops.workspace().f64("pcfactor", (2 * 148 + 8) * k * k + k * k + 1024)
    _lib.check(_lib.lib().gp_precond_factor(n, k, _lib.ptr(L), L.stride(0), float(noise),
                                            _lib.ptr(chol), _lib.ptr(binv), _lib.ptr(out),
                                            _lib.ptr(info), _lib.ptr(part), part.numel(),
                                            _lib.stream_handle()), "gp_precond_factor")
    host = D.to_host(T.cat([out, info.to(T.float64)]))   # one device->host read
    vals = host[:2]
    if int(host[2]) != 0 or not np.all(np.isfinite(vals)):
        raise NumericError("inner factorization of the preconditioner failed; "
                           "the factor is non-finite or the noise is not positive")
    return PreconditionerCache(L, noise, chol, binv, (n - k) * math.log(noise) + vals[0], vals[1])


def precond_apply_device(cache: PreconditionerCache, V):
    """P^{-1} V = (V - L B^{-1} L^T V) / noise on the device."""
    if cache.rank == 0:
        return V / cache.noise
    c = _ops.lowrank_mul(cache.binv_device, _ops.lt_mul(cache.factor_device, V))
    Y = V.clone()
    return _ops.lowrank_mul(cache.factor_device, c, Y, alpha=-1.0 / cache.noise,
                            beta=1.0 / cache.noise)


def precond_apply(cache: PreconditionerCache, V):
    """P^{-1} V via Woodbury (precond.py:125-139)."""
    Vd = D.to_device(V)
    squeeze = Vd.dim() == 1
    if squeeze:
        Vd = Vd[:, None]
    if Vd.shape[0] != cache.n:
        raise ValueError(f"V has {Vd.shape[0]} rows, preconditioner expects {cache.n}")
    out = D.to_host(precond_apply_device(cache, Vd.contiguous()))
    return out[:, 0] if squeeze else out


def precond_matmul(cache: PreconditionerCache, V):
    """P V (precond.py:142-147)."""
    Vd = D.to_device(V)
    squeeze = Vd.dim() == 1
    if squeeze:
        Vd = Vd[:, None]
    if cache.rank == 0:
        out = cache.noise * Vd
    else:
        out = _ops.lowrank_mul(cache.factor_device, _ops.lt_mul(cache.factor_device, Vd),
                               Vd.clone(), alpha=1.0, beta=cache.noise)
    out = D.to_host(out)
    return out[:, 0] if squeeze else out


def precond_sample_device(cache: PreconditionerCache, rng: np.random.Generator, t: int, draws=None):
    """Z = L z1 + sqrt(noise) z2 with z1 (k x t) drawn before z2 (n x t)
    from the host generator (precond.py:150-162) — bit-identical probes.
    `draws` = (z1, z2) already taken from a generator in that order."""
    if draws is None:
        z1 = rng.standard_normal((cache.rank, t))
        z2 = rng.standard_normal((cache.n, t))
    else:
        z1, z2 = draws
    z2 = D.to_device(z2)
    if cache.rank == 0:
        return math.sqrt(cache.noise) * z2
    return _ops.lowrank_mul(cache.factor_device, D.to_device(z1), z2, alpha=1.0,
                            beta=math.sqrt(cache.noise))


def precond_sample(cache: PreconditionerCache, rng: np.random.Generator, t: int) -> np.ndarray:
    return D.to_host(precond_sample_device(cache, rng, t))


def precond_inverse_quadratic_trace(cache: PreconditionerCache) -> float:
    """tr(P^{-1}) = (n - (k - noise tr B^{-1})) / noise (precond.py:165-174)."""
    if cache.rank == 0:
        return cache.n / cache.noise
    return (cache.n - (cache.rank - cache.noise * cache.tr_binv)) / cache.noise


def precond_weighted_trace(cache: PreconditionerCache, GL, trace_G: float) -> float:
    """tr(P^{-1} G) = (tr G - tr(B^{-1} L^T G L)) / noise (precond.py:177-185)."""
    if cache.rank == 0:
        return trace_G / cache.noise
    M = _ops.lt_mul(cache.factor_device, D.to_device(GL))
    tr = float((cache.binv_device * M.T).sum().item())
    return (trace_G - tr) / cache.noise
