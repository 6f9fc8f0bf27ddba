"""Row-sharded MLL + gradients and predictive mean across GPUs (one process
per GPU, torch.distributed) — SURVEY §8(e).

Rank r owns rows [row0, row1) of every CG block; X, y, the probe block Z and
the rank-k preconditioner are replicated (O(nd + nk) per GPU, as in the
paper). K̂·P runs the symmetric kernel with its work items
(unordered tile pairs) split across the ranks: each rank computes 64-bit
fixed-point partial sums for all rows, the int64 sums are all-reduced and
each rank finalises its rows (bitwise equal to the single-GPU product).
Exchanges:

* mBCG: all-gather of the fp32 search directions, all-reduce of the int64
  K̂·P partial sums (8 n t bytes) and of the fp64 reduction payload each
  iteration (cg.MbcgRun with a TorchComm);
* MLL: all-reduce of the local y·a partial; the SLQ log-determinant comes
  from the all-reduced alpha/beta histories, identical on every rank;
* gradients: all-gather of the representer weights a (8 n bytes), then each
  rank runs the fused gradient pass on its rows against all columns and the
  1 + n_l + 2 partial sums are all-reduced (likelihood.py:166-216);
* predictive mean: each rank contracts K(X*, X_local) a_local and the m test
  outputs are all-reduced (predictor.py:113-132);
* prediction cache: the representer-weight solve runs row-sharded like the
  MLL's, the weights are all-gathered (8 n bytes) (predictor.py:59-97);
* predictive variance: each 256-point chunk's batched solve runs row-sharded
  (rank r forms its rows of K(X, X*)), the m quadratic forms are all-reduced
  (predictor.py:135-182).

Under torch.distributed with world > 1 the reference-API entry points
(likelihood.mll_value_and_grad, predictor.build_cache / predict_mean /
predict_variance) dispatch here by themselves (distributed.active_comm).
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _ops
from . import precond as _pc
from .cg import FusedOperator, FusedOperator64, mbcg_device, slq_logdet
from .distributed import TorchComm
from .errors import NumericError
from .kernels import KernelModel
from .likelihood import (LOG_TWO_PI, CgConfig, MLLDiagnostics, MLLResult, _grad_forms_raw,
                         assemble_gradients, build_kernel_preconditioner, draw_probes_device)


def _local_gradient_operands(a_loc, S_loc, W_loc, a_full, W_full, cache, r0, r1):
    """Y rows of this shard and R over all rows for the fused gradient pass
    (same identity as likelihood.gradient_operands)."""
    T = D.torch()
    t = W_loc.shape[1]
    if cache is not None:
        Yc = [0.5 * a_loc[:, None], -(S_loc - W_loc) / (2.0 * t)]
        Rc = [a_full[:, None], W_full]
        if cache.rank:
            L = cache.factor_device
            Yc.append(_ops.lowrank_mul(L[r0:r1].contiguous(), cache.binv_device) / (2.0 * cache.noise))
            Rc.append(L)
    else:
        Yc = [0.5 * a_loc[:, None], -S_loc / (2.0 * t)]
        Rc = [a_full[:, None], W_full]
    Y = T.cat(Yc, dim=1).to(T.float32).contiguous()
    R = T.cat(Rc, dim=1).to(T.float32).contiguous()
    return Y, R


def mll_value_and_grad_sharded(model: KernelModel, X, y, cg_config: CgConfig, probe_seed: int,
                               comm: TorchComm) -> MLLResult:
    """mll_value_and_grad (likelihood.py:104-163) with K̂ rows sharded over
    the ranks of `comm`; every rank returns the same result."""
    T = D.torch()
    ps = D.points(X)
    n = ps.n
    if comm.n_total != n:
        raise ValueError("communicator was built for a different training size")
    yd = D.to_device(y)
    if tuple(yd.shape) != (n,):
        raise ValueError(f"y has shape {tuple(yd.shape)}, expected ({n},)")
    model.scale_for(ps.d)
    r0, r1 = comm.row0, comm.row1
    t = cg_config.probes
    yc = yd - model.mean
    cache = build_kernel_preconditioner(model, ps, cg_config.precond_rank)   # identical on every rank
    Z = draw_probes_device(n, t, probe_seed, cache)                          # identical on every rank
    Xs32, Xs64 = ps.scaled(model.scale_for(ps.d))
    if cg_config.precision == "fp64":   # this rank's rows of the fp64 operator
        op = FusedOperator64(_ops.Kv64Operator(model.family_code, ps.d, Xs64[r0:r1], Xs64, model.outputscale),
                             model.noise, n)
    else:
        # symmetric schedule split across the ranks (row-tiled kernel for t > 16)
        kv = _ops.training_operator(model.family_code, ps.d, Xs32, model.outputscale, 0.0, -1, comm)
        op = FusedOperator(kv, model.noise, n)
    B = T.cat([yc[:, None], Z], dim=1)[r0:r1].contiguous()
    sol = mbcg_device(op, B, cg_config.tolerance, cg_config.max_iters, cache, comm=comm, row_offset=r0)
    a_loc = sol.U[:, 0].contiguous()
    S_loc = sol.U[:, 1:].contiguous()
    logdet = slq_logdet(sol, cache, columns=range(1, t + 1), n_total=n)
    red = T.stack([_ops.coldot(yc[r0:r1, None].contiguous(), a_loc[:, None])[0], a_loc.sum()])
    comm.allreduce_(red)
    quad, asum = (float(v) for v in D.to_host(red))
    value = -0.5 * quad - 0.5 * logdet - 0.5 * n * LOG_TWO_PI
    W_full = _pc.precond_apply_device(cache, Z) if cache is not None else Z
    W_loc = W_full[r0:r1].contiguous()
    a_full = T.zeros(comm.rows_per_rank * comm.world, dtype=T.float64, device=a_loc.device)
    a_pad = T.zeros(comm.rows_per_rank, dtype=T.float64, device=a_loc.device)
    a_pad[: r1 - r0] = a_loc
    comm.allgather_rows(a_pad, a_full)
    a_full = a_full[:n].contiguous()
    Y, R = _local_gradient_operands(a_loc, S_loc, W_loc, a_full, W_full, cache, r0, r1)
    raw = _grad_forms_raw(model, ps.d, Xs32[r0:r1], Xs32, Y, R, self_offset=r0)
    gradients = assemble_gradients(model, raw, a_loc, S_loc, W_loc, cache, n,
                                   reduce=lambda v: comm.allreduce_(v.contiguous()))
    gradients["mean"] = asum
    if not np.isfinite(value) or any(not np.isfinite(g) for g in gradients.values()):
        raise NumericError("non-finite likelihood value or gradient")
    diag = MLLDiagnostics(probe_seed=probe_seed, iterations=sol.iterations, final_residuals=sol.rel,
                          converged=bool(sol.converged.all()), logdet_estimate=logdet, quad_term=quad,
                          precond_rank=cache.rank if cache is not None else 0)
    return MLLResult(value=value, gradients=gradients, diagnostics=diag)


def _allgather_vector(local, comm: TorchComm, n: int):
    """The full n-vector from each rank's rows (all-gather of the padded
    slices)."""
    T = D.torch()
    m = comm.rows_per_rank
    pad = T.zeros(m, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    full = T.zeros(m * comm.world, dtype=local.dtype, device=local.device)
    comm.allgather_rows(pad, full)
    return full[:n].contiguous()


def build_cache_sharded(model: KernelModel, X, y, comm: TorchComm, *, tolerance: float = 1e-3,
                        max_iters: int = 1000, precond_rank: int = 100):
    """build_cache (predictor.py:59-97) with the representer-weight solve
    row-sharded over the ranks of `comm` (the paper's one-time 'precompute'
    of the predictive cache); every rank returns the same PredictionCache."""
    from .errors import ConvergenceError
    from .predictor import PredictionCache
    ps = D.points(X)
    n = ps.n
    if comm.n_total != n:
        raise ValueError("communicator was built for a different training size")
    yd = D.to_device(y)
    if tuple(yd.shape) != (n,):
        raise ValueError(f"y has shape {tuple(yd.shape)}, expected ({n},)")
    r0, r1 = comm.row0, comm.row1
    cache_p = build_kernel_preconditioner(model, ps, precond_rank)   # identical on every rank
    Xs32, _ = ps.scaled(model.scale_for(ps.d))
    kv = _ops.training_operator(model.family_code, ps.d, Xs32, model.outputscale, 0.0, -1, comm)
    op = FusedOperator(kv, model.noise, n)
    B = (yd - model.mean)[r0:r1, None].contiguous()
    sol = mbcg_device(op, B, tolerance, max_iters, cache_p, comm=comm, row_offset=r0)
    if not sol.converged.all():
        raise ConvergenceError(
            f"representer-weight solve stalled at relative residual {float(sol.rel[0]):.3e} "
            f"(requested {tolerance:g})", residuals=sol.rel)
    w_dev = _allgather_vector(sol.U[:, 0].contiguous(), comm, n)
    pc = PredictionCache(model=model, X_train=X if not D.is_tensor(X) else D.to_host(X),
                         weights=D.to_host(w_dev), cache_tolerance=tolerance,
                         diagnostics={"iterations": sol.iterations, "residual": float(sol.rel[0]),
                                      "precond_rank": precond_rank})
    pc._w_dev = w_dev
    return pc


def predict_mean_sharded(model: KernelModel, X_train, weights, X_test, comm: TorchComm,
                         precision: str = "fp64") -> np.ndarray:
    """mu + K(X*, X) a with the training columns sharded: each rank contracts
    its columns, the m test outputs are all-reduced (predictor.py:113-132).
    fp64 (gp_kv_f64) by default, like the single-device predict_mean."""
    T = D.torch()
    tr = D.points(X_train)
    te = D.points(np.atleast_2d(X_test) if not D.is_tensor(X_test) else X_test)
    if te.d != tr.d:
        raise ValueError(f"test points have dimension {te.d}, training data has {tr.d}")
    r0, r1 = comm.row0, comm.row1
    ls = model.scale_for(tr.d)
    Xr32, Xr64 = te.scaled(ls)
    Xc32, Xc64 = tr.scaled(ls)
    w = D.to_device(weights)[r0:r1].contiguous()
    if precision == "fp64":
        part, _ = _ops.kv_f64(model.family_code, tr.d, Xr64, Xc64[r0:r1], model.outputscale, 0.0, -1, w)
        part = part[:, 0].contiguous()
    else:
        kv = _ops.FusedKernelOperator(model.family_code, tr.d, Xr32, Xc32[r0:r1], model.outputscale, 0.0, -1)
        part = kv.apply32(w[:, None].to(T.float32).contiguous(), 1)[:, 0].to(T.float64).contiguous()
    comm.allreduce_(part)
    return model.mean + D.to_host(part)


def predict_variance_sharded(cache, X_test, comm: TorchComm, *, tolerance: float = 0.01,
                             max_iters: int = 1000, precond_rank: int = 100, chunk: int = 256):
    """predict_variance (predictor.py:135-182) with every batched solve
    row-sharded: rank r forms its rows of B = K(X, X*_chunk), the solve runs
    over all ranks (t = chunk right-hand sides: the row-tiled wide kernel on
    this rank's rows against the all-gathered directions), and the
    quadratic forms colsum(B o S) are all-reduced. Every rank returns the same
    (variances, clamped)."""
    from .errors import ConvergenceError
    from .kernels import _dense_block
    X_test = np.atleast_2d(X_test) if not D.is_tensor(X_test) else X_test
    model = cache.model
    tr = D.points(cache.X_train)
    n = tr.n
    if X_test.shape[1] != tr.d:
        raise ValueError("test/train dimension mismatch")
    if comm.n_total != n:
        raise ValueError("communicator was built for a different training size")
    r0, r1 = comm.row0, comm.row1
    cache_p = build_kernel_preconditioner(model, tr, precond_rank)
    Xs32, _ = tr.scaled(model.scale_for(tr.d))
    kv = _ops.training_operator(model.family_code, tr.d, Xs32, model.outputscale, 0.0, -1, comm)
    op = FusedOperator(kv, model.noise, n)
    m = X_test.shape[0]
    out = np.empty(m)
    clamped = 0
    for c0 in range(0, m, chunk):
        c1 = min(c0 + chunk, m)
        te = D.points(X_test[c0:c1])
        Bm = _dense_block(model, tr, te, -1, (r0, r1)).contiguous()
        sol = mbcg_device(op, Bm, tolerance, max_iters, cache_p, comm=comm, row_offset=r0)
        if not sol.converged.all():
            bad = np.flatnonzero(~sol.converged)
            raise ConvergenceError(f"variance solves for {bad.size} test points did not reach "
                                   f"tolerance {tolerance:g}", residuals=sol.rel)
        quad = comm.allreduce_(_ops.coldot(Bm, sol.U))
        var = model.outputscale - D.to_host(quad)
        low = var < 1e-12
        clamped += int(np.count_nonzero(low))
        var[low] = 1e-12
        out[c0:c1] = var
    return out, clamped
