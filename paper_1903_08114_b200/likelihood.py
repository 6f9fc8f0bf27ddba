"""Exact-GP log marginal likelihood and gradients (mirror of blockgp.likelihood).

One device-resident mBCG solve over [y - mu | Z] (probes Z drawn with
covariance P from the host generator, bit-identical to the reference),
SLQ on the probe columns for logdet, and ONE fused gradient pass
(gp_grad_forms) for every geometric hyperparameter:

    g_p = sum_ij (dK/dtheta_p)_ij (Y R^T)_ij - tr(dK/dtheta_p) / (2 noise)
    Y = [a/2 | -(S-W)/(2t) | L B^{-1}/(2 noise)],   R = [a | W | L]

which is algebraically identical to the reference's per-parameter products
(likelihood.py:166-216; identity derived in SURVEY §7.3(6)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from . import _ops
from . import precond as _pc
from .cg import FusedOperator, FusedOperator64, mbcg_device, slq_logdet
from .distributed import active_comm
from .errors import NumericError
from .kernels import KernelModel, param_ids
from .partition import PartitionPlan, WorkerPool

LOG_TWO_PI = math.log(2.0 * math.pi)


@dataclass
class CgConfig:
    """Training-protocol solver settings (likelihood.py:38-54)."""

    tolerance: float = 1.0
    max_iters: int = 1000
    probes: int = 10
    precond_rank: int = 100
    # operator precision of the mBCG solve: "fp32" = the tcgen05 K·V kernels
    # (north_star tolerance, SFU-bound); "fp64" = gp_kv_f64, the reference's
    # float64 operator. The loose-tolerance (eps = 1) solves of the training
    # protocol are a chaotic function of operator round-off once CG runs for
    # tens of iterations (C2: 37 iterations in fp64, 43 with the ~1e-6 fp32
    # operator), so "fp64" is what reproduces the reference's iteration
    # counts and values there (tests/test_gpu_large_configs.py).
    precision: str = "fp32"

    def __post_init__(self):
        if self.probes < 1:
            raise ValueError("at least one probe vector is required")
        if self.precision not in ("fp32", "fp64"):
            raise ValueError(f"precision must be 'fp32' or 'fp64', got {self.precision!r}")


@dataclass
class MLLDiagnostics:
    probe_seed: int
    iterations: int
    final_residuals: np.ndarray
    converged: bool
    logdet_estimate: float
    quad_term: float
    precond_rank: int


@dataclass
class MLLResult:
    value: float
    gradients: dict
    diagnostics: MLLDiagnostics = field(repr=False)


def build_kernel_preconditioner(model: KernelModel, X, rank: int, overlap=None):
    """Rank-min(rank, n) pivoted-Cholesky preconditioner of the noiseless
    kernel (likelihood.py:74-91); None when rank <= 0. `overlap` runs on the
    host while the device factorises."""
    if rank <= 0:
        return None
    src = _pc.KernelRowSource(model, X)
    n = src.points.n
    k = min(rank, n)
    factor = _pc.partial_pivoted_cholesky(src, np.full(n, model.outputscale), k, overlap)
    return _pc.build_preconditioner(factor, model.noise)


def draw_probes_device(n: int, t: int, seed: int, cache, draws=None):
    """`draws`: the (z1, z2) normals already taken from default_rng(seed) for
    a rank-`cache.rank` preconditioner (drawn while the factor was built)."""
    rng = np.random.default_rng(seed)
    if cache is None:   # z1 is empty: z2 is the stream's first n x t normals
        return D.to_device(draws[1] if draws is not None else rng.standard_normal((n, t)))
    if draws is not None and draws[0].shape[0] != cache.rank:
        draws = None   # the factorisation stopped early: the z2 stream position differs
    return _pc.precond_sample_device(cache, rng, t, draws)


class ProbeDraws:
    """The seeded probes' host normals (likelihood.py:94-101: z1 = k x t,
    then z2 = n x t, from default_rng(seed)), bit-identical to the reference.
    Large blocks (>= 2^20 normals) are drawn on a helper thread started
    before the inputs are uploaded, so the draw overlaps the upload, the
    prescale and the pivoted Cholesky (numpy's generator fills without the
    GIL); small ones are drawn inline while the device factorises."""

    THREAD_MIN = 1 << 20

    def __init__(self, seed: int, k: int, n: int, t: int):
        self.args = (seed, k, n, t)
        self.out = None
        self.thread = None
        if n * t >= self.THREAD_MIN:
            import threading
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()

    def _run(self):
        seed, k, n, t = self.args
        rng = np.random.default_rng(seed)
        z1 = rng.standard_normal((k, t))
        self.out = (z1, rng.standard_normal((n, t)))

    def overlap(self):
        """Host work to run while the device factorises (the inline case)."""
        if self.thread is None and self.out is None:
            self._run()

    def result(self):
        """(z1, z2), or None if the draw failed (the caller then draws)."""
        if self.thread is not None:
            self.thread.join()
        elif self.out is None:
            self._run()
        return self.out


def draw_probes(n: int, t: int, seed: int, cache) -> np.ndarray:
    """Seeded probes: N(0, I) or N(0, P) (likelihood.py:94-101)."""
    return D.to_host(draw_probes_device(n, t, seed, cache))


def training_operator(model: KernelModel, ps, algo: int = 0, precision: str = "fp32", workers: int = 1,
                      t: int = 1):
    """K̂ as the mBCG operator. `workers` > 1 (a WorkerPool's thread count,
    partition.py:46-57) spans that many GPUs of this process when the host
    has them (multidev.py); `t` is the right-hand-side count it will see."""
    Xs32, Xs64 = ps.scaled(model.scale_for(ps.d))
    if precision == "fp64":
        return FusedOperator64(_ops.Kv64Operator(model.family_code, ps.d, Xs64, Xs64, model.outputscale),
                               model.noise, ps.n)
    kv = _ops.FusedKernelOperator(model.family_code, ps.d, Xs32, Xs32, model.outputscale, 0.0,
                                  -1, algo=algo, self_offset=0)
    if workers > 1 and algo == 0:
        from .multidev import training_operator as multi
        kv = multi(model.family_code, ps.d, Xs32, model.outputscale, 0.0, -1, workers, t, kv)
    return FusedOperator(kv, model.noise, ps.n)


def mll_value_and_grad(model: KernelModel, X, y, plan: PartitionPlan, pool: WorkerPool,
                       cg_config: CgConfig, probe_seed: int) -> MLLResult:
    """log p(y) and d/dtheta for every trainable hyperparameter
    (likelihood.py:104-163), computed on the GPU."""
    T = D.torch()
    n0 = X.n if isinstance(X, D.PointSet) else len(X)
    k0 = min(cg_config.precond_rank, n0) if cg_config.precond_rank > 0 else 0
    # started before the upload; the sharded path below draws its own
    draws = ProbeDraws(probe_seed, k0, n0, cg_config.probes) if active_comm(n0) is None else None
    ps = D.points(X)
    n = ps.n
    yd = D.to_device(y)
    if tuple(yd.shape) != (n,):
        raise ValueError(f"y has shape {tuple(yd.shape)}, expected ({n},)")
    if plan.n != n:
        raise ValueError("partition plan does not match the training size")
    model.scale_for(ps.d)
    comm = active_comm(n)
    if comm is not None:  # under torchrun: rows sharded over the ranks
        from .sharded import mll_value_and_grad_sharded
        return mll_value_and_grad_sharded(model, ps, yd, cg_config, probe_seed, comm)
    t = cg_config.probes
    yc = yd - model.mean
    # the probes' host normals (likelihood.py:94-101) come from ProbeDraws:
    # a helper thread for large n, else drawn while the device factorises
    cache = build_kernel_preconditioner(model, ps, cg_config.precond_rank, overlap=draws.overlap)
    Z = draw_probes_device(n, t, probe_seed, cache, draws.result())
    op = training_operator(model, ps, precision=cg_config.precision, workers=pool.workers, t=t + 1)
    B = T.cat([yc[:, None], Z], dim=1).contiguous()
    sol = mbcg_device(op, B, cg_config.tolerance, cg_config.max_iters, cache)
    a = sol.U[:, 0].contiguous()
    S = sol.U[:, 1:].contiguous()
    # y^T a and sum(a) stay on the device until the gradients' read
    qa_dev = T.stack([_ops.coldot(yc[:, None], a[:, None])[0], a.sum()])
    logdet = slq_logdet(sol, cache, columns=range(1, t + 1))
    W = _pc.precond_apply_device(cache, Z) if cache is not None else Z
    gradients = _gradients(model, ps, a, S, W, cache)
    qa = D.to_host(qa_dev)
    quad = float(qa[0])
    value = -0.5 * quad - 0.5 * logdet - 0.5 * n * LOG_TWO_PI
    gradients["mean"] = float(qa[1])
    if not np.isfinite(value) or any(not np.isfinite(g) for g in gradients.values()):
        raise NumericError("non-finite likelihood value or gradient")
    diag = MLLDiagnostics(probe_seed=probe_seed, iterations=sol.iterations,
                          final_residuals=sol.rel, converged=bool(sol.converged.all()),
                          logdet_estimate=logdet, quad_term=quad,
                          precond_rank=cache.rank if cache is not None else 0)
    return MLLResult(value=value, gradients=gradients, diagnostics=diag)


def gradient_operands(a, S, W, cache):
    """fp32 (Y, R) of the fused gradient pass, plus the constant
    tr(dK/ds2)/(2 noise) to subtract from the outputscale form."""
    T = D.torch()
    t = W.shape[1]
    if cache is not None:
        Yc = [0.5 * a[:, None], -(S - W) / (2.0 * t)]
        Rc = [a[:, None], W]
        if cache.rank:
            LB = _ops.lowrank_mul(cache.factor_device, cache.binv_device)
            Yc.append(LB / (2.0 * cache.noise))
            Rc.append(cache.factor_device)
    else:
        Yc = [0.5 * a[:, None], -S / (2.0 * t)]
        Rc = [a[:, None], W]
    Y = T.cat(Yc, dim=1).to(T.float32).contiguous()
    R = T.cat(Rc, dim=1).to(T.float32).contiguous()
    return Y, R


def symmetric_gradient_operands(a, S, W, cache):
    """fp32 (Y_s, R_s) with Y_s R_s^T = (H + H^T)/2 for the H = Y R^T of
    gradient_operands: only the probe block is asymmetric, so it appears
    twice with half the weight. Every dK/dtheta is symmetric, so the forms
    against H_s equal those against H while the kernel sums each unordered
    pair of points once (gp_grad_forms_sym)."""
    T = D.torch()
    t = W.shape[1]
    if cache is not None:
        D_ = S - W
        Yc = [0.5 * a[:, None], -D_ / (4.0 * t), -W / (4.0 * t)]
        Rc = [a[:, None], W, D_]
        if cache.rank:
            LB = _ops.lowrank_mul(cache.factor_device, cache.binv_device)
            Yc.append(LB / (2.0 * cache.noise))
            Rc.append(cache.factor_device)
    else:
        Yc = [0.5 * a[:, None], -S / (4.0 * t), -W / (4.0 * t)]
        Rc = [a[:, None], W, S]
    Y = T.cat(Yc, dim=1).to(T.float32).contiguous()
    R = T.cat(Rc, dim=1).to(T.float32).contiguous()
    return Y, R


def _grad_forms_sym_raw(model, d, Xs32, Y, R):
    """Raw forms over the square operator with the symmetric schedule
    (csrc/grad_tc.cu, gp_grad_forms_sym)."""
    T = D.torch()
    ard = 1 if model.ard else 0
    npar = 1 + (d if ard else 1)
    out = T.zeros(npar, dtype=T.float64, device=D.device())
    lib = _lib.lib()
    n, w = Xs32.shape[0], Y.shape[1]
    nbytes = lib.gp_grad_forms_sym_workspace_bytes(n, d, ard, w)
    ws = _ops.workspace().bytes("grad", nbytes)
    _lib.check(lib.gp_grad_forms_sym(model.family_code, d, ard, _lib.ptr(Xs32), Xs32.stride(0), n,
                                     float(model.outputscale), _lib.ptr(Y), Y.stride(0), _lib.ptr(R),
                                     R.stride(0), w, _lib.ptr(out), _lib.ptr(ws), nbytes,
                                     _lib.stream_handle()), "gp_grad_forms_sym")
    return out


def _gradients(model: KernelModel, ps, a, S, W, cache) -> dict:
    n, t = W.shape
    Xs32, _ = ps.scaled(model.scale_for(ps.d))
    k = cache.rank if cache is not None else 0
    w_sym = 1 + 2 * t + k
    if _lib.lib().gp_grad_forms_sym_supported(n, ps.d, 1 if model.ard else 0, w_sym):
        # each unordered pair of points once (the per-entry tcgen05 kernel)
        Y, R = symmetric_gradient_operands(a, S, W, cache)
        raw = _grad_forms_sym_raw(model, ps.d, Xs32, Y, R)
    else:
        # large d (e.g. C4, d = 90): the full square with the narrower
        # non-symmetric operands (w = 1 + t + k), which the tensor-core ARD
        # expansion takes (csrc/grad_ard.cu, w <= 112)
        Y, R = gradient_operands(a, S, W, cache)
        raw = _grad_forms_raw(model, ps.d, Xs32, Xs32, Y, R)
    return assemble_gradients(model, raw, a, S, W, cache, n)


def _grad_forms_raw(model, d, Xr32, Xc32, Y, R, self_offset=0, algo=0):
    """Raw fused gradient forms (csrc/grad_tc.cu, csrc/grad.cu); row i of
    Xr32 is column i + self_offset of Xc32."""
    T = D.torch()
    ard = 1 if model.ard else 0
    npar = 1 + (d if ard else 1)
    out = T.zeros(npar, dtype=T.float64, device=D.device())
    lib = _lib.lib()
    w = Y.shape[1]
    nbytes = lib.gp_grad_forms_workspace_bytes(Xr32.shape[0], Xc32.shape[0], d, ard, w)
    ws = _ops.workspace().bytes("grad", nbytes)
    _lib.check(lib.gp_grad_forms(model.family_code, d, ard, _lib.ptr(Xr32), Xr32.stride(0),
                                 Xr32.shape[0], _lib.ptr(Xc32), Xc32.stride(0), Xc32.shape[0],
                                 float(model.outputscale), _lib.ptr(Y), Y.stride(0), _lib.ptr(R),
                                 R.stride(0), w, int(self_offset), int(algo), _lib.ptr(out),
                                 _lib.ptr(ws), nbytes, _lib.stream_handle()), "gp_grad_forms")
    return out


def assemble_gradients(model, raw_dev, a, S, W, cache, n_total: int, reduce=None) -> dict:
    """Constant factors + noise gradient (likelihood.py:192-216). `reduce`
    all-reduces device scalars when rows are sharded."""
    T = D.torch()
    t = W.shape[1]
    # device scalars: [a.a, sum (S-W) o W  (or S o W)]
    if cache is not None:
        sw = _ops.coldot((S - W).contiguous(), W).sum()
    else:
        sw = _ops.coldot(S, W).sum()
    aa = _ops.coldot(a[:, None], a[:, None])[0]
    vec = T.cat([raw_dev, aa[None], sw[None]])
    if reduce is not None:
        vec = reduce(vec)
    v = D.to_host(vec)
    raw, aa, sw = v[:-2], float(v[-2]), float(v[-1])
    s2 = model.outputscale
    g = {}
    const = 0.5 * n_total / cache.noise if cache is not None else 0.0
    g["outputscale"] = float(raw[0]) - const
    if model.ard:
        for i, l in enumerate(model.lengthscales):
            g[f"lengthscale_{i}"] = s2 * float(raw[1 + i]) / float(l)
    else:
        g["lengthscale"] = s2 * float(raw[1]) / float(model.lengthscales[0])
    if cache is not None:
        tr_noise = _pc.precond_inverse_quadratic_trace(cache) if n_total == cache.n else \
            (n_total - (cache.rank - cache.noise * cache.tr_binv)) / cache.noise
        g["noise"] = 0.5 * aa - 0.5 * (tr_noise + sw / t)
    else:
        g["noise"] = 0.5 * aa - 0.5 * sw / t
    ordered = {}
    for pid in param_ids(model):
        if pid in g:
            ordered[pid] = g[pid]
    return ordered
