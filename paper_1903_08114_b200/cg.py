"""Batched preconditioned CG with Lanczos coefficients (mirror of blockgp.cg).

The solve runs device-resident through the gp_mbcg_* phases of the C-ABI
(cg.py:84-164 semantics: per-column freeze on the recurrence residual
||r||/||b||, alpha/beta recorded for active columns only). The host reads
one small status word per iteration to decide termination; the alpha/beta
history stays in HBM until the end. SLQ (cg.py:182-218) runs on the host on
the t tiny tridiagonals, as in the reference.

Operators (`mvm`):
  * a fused kernel operator (likelihood/predictor build them): K·P on
    gp_kv from the fp32 copy of P, noise*P added in fp64 by the CG kernels;
  * any callable on (n, j) arrays (numpy in/out, or CUDA tensors in/out):
    applied to the active columns, fp64 end to end.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from . import _ops
from .errors import NumericError
from .precond import PreconditionerCache


@dataclass
class SolveRequest:
    """rhs columns, relative-residual tolerance, iteration cap, optional
    preconditioner (cg.py:27-49)."""

    rhs: object
    tolerance: float
    max_iters: int = 1000
    preconditioner: PreconditionerCache | None = None

    def __post_init__(self):
        if D.is_tensor(self.rhs):
            r = self.rhs
            if r.dim() == 1:
                r = r[:, None]
            if r.dim() != 2:
                raise ValueError("rhs must be a vector or a matrix of columns")
            self.rhs = r
            norms = D.to_host(D.torch().linalg.norm(r.to(D.torch().float64), dim=0))
        else:
            r = np.asarray(self.rhs, dtype=np.float64)
            if r.ndim == 1:
                r = r[:, None]
            if r.ndim != 2:
                raise ValueError("rhs must be a vector or a matrix of columns")
            self.rhs = r
            norms = np.linalg.norm(r, axis=0)
        if not self.tolerance > 0:
            raise ValueError(f"tolerance must be positive, got {self.tolerance}")
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if np.any(norms == 0):
            raise ValueError("every right-hand-side column must be non-zero")


@dataclass(frozen=True)
class Tridiagonal:
    """Lanczos matrix of one column (cg.py:52-69)."""

    diag: np.ndarray
    offdiag: np.ndarray

    @property
    def order(self) -> int:
        return self.diag.shape[0]

    def dense(self) -> np.ndarray:
        T = np.diag(self.diag)
        if self.offdiag.size:
            i = np.arange(self.offdiag.size)
            T[i, i + 1] = self.offdiag
            T[i + 1, i] = self.offdiag
        return T


@dataclass
class SolveReport:
    solutions: np.ndarray
    final_relative_residuals: np.ndarray
    iterations: int
    tridiagonals: list
    converged: np.ndarray
    residual_history: np.ndarray = field(repr=False)
    solutions_device: object = field(default=None, repr=False)


class FusedOperator:
    """K̂ = s2 kappa(X, X) + noise I applied by gp_kv on this device's rows.
    `apply32(P32_full, t, out32)` computes the noiseless K·P; the CG kernels
    add noise*P in fp64."""

    fused = True

    def __init__(self, kv_op: _ops.FusedKernelOperator, noise: float, n_total: int,
                 gather=None):
        self.kv = kv_op
        self.noise = float(noise)
        self.n_total = n_total
        self.gather = gather  # distributed: all-gather of the local P32 rows

    def __call__(self, V):  # reference-style use
        T = D.torch()
        Vd = D.to_device(V)
        out = self.kv.apply32(Vd.to(T.float32).contiguous(), Vd.shape[1]).to(T.float64)
        out += self.noise * Vd
        return out if D.is_tensor(V) else D.to_host(out)


class FusedOperator64:
    """K̂ = s2 kappa(X, X) + noise I with the kernel part applied in fp64
    (gp_kv_f64) on this device's rows: the precision of the reference's
    partitioned_mvm (float64 end to end). `apply64(P64_full, t, out64)`
    computes the noiseless K·P; the CG kernels add noise*P in fp64."""

    fused = True
    f64 = True

    def __init__(self, kv64, noise: float, n_total: int):
        self.kv = kv64
        self.noise = float(noise)
        self.n_total = n_total

    def __call__(self, V):
        Vd = D.to_device(V)
        if Vd.dim() == 1:
            Vd = Vd[:, None]
        out = self.kv.apply64(Vd.contiguous(), Vd.shape[1]) + self.noise * Vd
        return out if D.is_tensor(V) else D.to_host(out)


def _tridiagonal(al, be) -> Tridiagonal:
    """cg.py:167-179: diag_i = 1/a_i + b_{i-1}/a_{i-1}, off_i = sqrt(b_i)/a_i."""
    m = len(al)
    diag = np.empty(m)
    off = np.empty(max(m - 1, 0))
    for i in range(m):
        diag[i] = 1.0 / al[i] + (be[i - 1] / al[i - 1] if i else 0.0)
        if i < m - 1:
            off[i] = math.sqrt(be[i]) / al[i]
    return Tridiagonal(diag=diag, offdiag=off)


class _Comm:
    """No-op communicator (single device)."""

    world = 1

    def allreduce_(self, t):
        return t

    def allgather_rows(self, local, full):
        full.copy_(local)
        return full


class DeviceSolve:
    """Result of a device-resident solve (tensors stay in HBM)."""

    def __init__(self, U, rel, iterations, alphas, betas, converged, history):
        self.U = U
        self.rel = rel
        self.iterations = iterations
        self.alphas = alphas
        self.betas = betas
        self.converged = converged
        self.history = history

    def tridiagonals(self):
        return [_tridiagonal(a, b) for a, b in zip(self.alphas, self.betas)]


_pinned = threading.local()


def _pinned_status():
    """A pinned 4 x int32 host buffer for the per-iteration status read,
    allocated once per thread (pinned allocations are slow)."""
    buf = getattr(_pinned, "status", None)
    if buf is None:
        buf = _pinned.status = D.torch().zeros(4, dtype=D.torch().int32).pin_memory()
    return buf


class CudaPhases:
    """The mBCG phase kernels of the C ABI (gp_mbcg_*) on this device's rows,
    owning the solver state in HBM. MbcgRun drives it; tests substitute a
    restatement with the same interface to exercise the sharded driver on CPU."""

    def __init__(self, n, t, k, max_iters, noise, precond, L_local, rows32):
        T = D.torch()
        self.T = T
        self.lib = _lib.lib()
        self.st = _lib.stream_handle()
        dev = D.device()
        self.n, self.t, self.k = n, t, k
        self.ld32 = ld32 = (t + 3) // 4 * 4
        f64 = dict(dtype=T.float64, device=dev)
        self.U = T.empty((n, t), **f64)   # the solution (handed to the caller)
        self.R, self.P, self.Z = T.empty((3, n, t), **f64).unbind(0)
        self.P32 = T.zeros((max(rows32, n), ld32), dtype=T.float32, device=dev)
        # the small state in one zero-filled allocation (one fill per solve)
        sizes = [3 * t + k * t, max(k * t, 1), 3 * max_iters * t, 3 * t, (2 * t + 4 + 1) // 2]
        small = T.zeros(sum(sizes), **f64)
        red, cbuf, hist, vec, ints = small.split(sizes)
        self.red, self.cbuf = red, cbuf
        self.hist = hist.view(3, max_iters, t)  # alpha, beta, rel
        self.vec = vec.view(3, t)  # bnorm, gamma, rel
        self.ints = ints.view(T.int32)[:2 * t + 4]
        plen = int(self.lib.gp_mbcg_partials_len(n, t, k))
        self.partials = _ops.workspace().f64("mbcg_partials", plen)
        self.state = _lib.MbcgState(
            n=n, t=t, k=k, ld=t, ld32=ld32, U=_lib.ptr(self.U), R=_lib.ptr(self.R),
            P=_lib.ptr(self.P), Z=_lib.ptr(self.Z), P32=_lib.ptr(self.P32), noise=float(noise),
            L=_lib.ptr(L_local) if k else 0, ldl=L_local.stride(0) if k else 0,
            Binv=_lib.ptr(precond.binv_device) if k else 0,
            pc_noise=float(precond.noise) if precond is not None else 0.0,
            bnorm=_lib.ptr(self.vec[0]), gamma=_lib.ptr(self.vec[1]), red=_lib.ptr(self.red),
            cbuf=_lib.ptr(self.cbuf), alpha_hist=_lib.ptr(self.hist[0]),
            beta_hist=_lib.ptr(self.hist[1]), rel=_lib.ptr(self.vec[2]),
            rel_hist=_lib.ptr(self.hist[2]), active=_lib.ptr(self.ints[:t]),
            converged=_lib.ptr(self.ints[t:2 * t]), status=_lib.ptr(self.ints[2 * t:]),
            partials=_lib.ptr(self.partials), partials_len=plen, max_iters=max_iters, nblocks=0)
        self.sp = _lib.C.byref(self.state)
        self.status_host = _pinned_status()

    def init_a(self, B):
        _lib.check(self.lib.gp_mbcg_init_a(self.sp, _lib.ptr(B), B.stride(0), self.st), "gp_mbcg_init_a")

    def init_b(self):
        _lib.check(self.lib.gp_mbcg_init_b(self.sp, self.st), "gp_mbcg_init_b")

    def init_c(self):
        _lib.check(self.lib.gp_mbcg_init_c(self.sp, self.st), "gp_mbcg_init_c")

    def pv(self, Q, q_f64):
        _lib.check(self.lib.gp_mbcg_pv(self.sp, _lib.ptr(Q), Q.stride(0), int(q_f64), self.st),
                   "gp_mbcg_pv")

    def update(self, Q, q_f64, it):
        _lib.check(self.lib.gp_mbcg_update(self.sp, _lib.ptr(Q), Q.stride(0), int(q_f64), it,
                                           self.st), "gp_mbcg_update")

    def precond(self, it, tol):
        _lib.check(self.lib.gp_mbcg_precond(self.sp, it, float(tol), self.st), "gp_mbcg_precond")

    def direction(self, it):
        _lib.check(self.lib.gp_mbcg_direction(self.sp, it, self.st), "gp_mbcg_direction")

    def active(self):
        return self.ints[:self.t]

    def zero_rhs_columns(self) -> bool:
        """True if some column of B has ||b|| = 0 (bnorm after init, global
        over ranks); one small device->host read per solve."""
        return bool(D.to_host((self.vec[0] == 0).any()))

    def status(self):
        """(active columns, first non-PD column or >= t, its iteration); syncs."""
        self.status_host.copy_(self.ints[2 * self.t:], non_blocking=True)
        self.T.cuda.current_stream().synchronize()
        s = self.status_host
        return int(s[0]), int(s[1]), int(s[2])

    def history(self, its):
        """(alpha/beta/rel history, final rel, converged) in one device->host read."""
        T, t = self.T, self.t
        flat = D.to_host(T.cat([self.hist[:, :its].reshape(-1), self.vec[2],
                                self.ints[t:2 * t].to(T.float64)]))
        h = 3 * its * t
        return flat[:h].reshape(3, its, t), flat[h:h + t].copy(), flat[h + t:] != 0


class MbcgRun:
    """Steppable device-resident mBCG (cg.py:84-164) on this device's rows.

    `step()` runs one iteration (K·P, alpha/U/R update, freeze, Z, beta/P)
    and returns the number of still-active columns; `finish()` folds the
    device-side alpha/beta/residual history into a DeviceSolve. With a
    multi-rank `comm`, the reduction payload is all-reduced between phases
    and the fp32 search directions are all-gathered before each K·P."""

    def __init__(self, mvm, B, tol: float, max_iters: int = 1000,
                 precond: PreconditionerCache | None = None, comm=None, row_offset: int = 0,
                 phases_factory=None):
        T = D.torch()
        self.T = T
        self.comm = comm or _Comm()
        B = B.to(T.float64).contiguous()
        n, t = B.shape
        self.n, self.t, self.tol, self.max_iters = n, t, float(tol), int(max_iters)
        self.mvm = mvm
        self.precond = precond
        k = precond.rank if precond is not None else 0
        self.k = k
        L = precond.factor_device if precond is not None else None
        if L is not None and L.shape[0] != n:
            L = L[row_offset:row_offset + n]
        self.fused = bool(getattr(mvm, "fused", False))
        rows32 = getattr(self.comm, "rows_per_rank", n) if self.comm.world > 1 else n
        factory = phases_factory or CudaPhases
        self.ph = factory(n, t, k, self.max_iters, float(mvm.noise) if self.fused else 0.0,
                          precond, L, rows32)
        self.U = self.ph.U
        self.f64 = self.fused and bool(getattr(mvm, "f64", False))
        if self.f64:
            P = self.ph.P
            self.Q = T.empty((n, t), dtype=T.float64, device=P.device)
            if self.comm.world > 1:
                self.P64_loc = T.zeros((rows32, t), dtype=T.float64, device=P.device)
                self.P64_full = T.zeros((rows32 * self.comm.world, t), dtype=T.float64, device=P.device)
        elif self.fused:
            P32 = self.ph.P32
            self.Q = T.empty((n, t), dtype=T.float32, device=P32.device)
            total = mvm.n_total if self.comm.world == 1 else rows32 * self.comm.world
            self.P32_full = P32 if self.comm.world == 1 else \
                T.zeros((total, P32.shape[1]), dtype=T.float32, device=P32.device)
        self.iterations = 0
        self.kv_events = None  # optional (start, end) CUDA events around K·P
        self.ph.init_a(B)
        self._allreduce(t, 2 * t + k * t)
        self.ph.init_b()
        self._allreduce(2 * t + k * t, 3 * t + k * t)
        self.ph.init_c()
        # cg.py:47-49: a zero right-hand-side column is an argument error
        # (ValueError), whichever caller built the block (SolveRequest, the
        # MLL's [y - mu | Z], or the variance solve's cross-kernel columns
        # of a test point far from every training point)
        if self.ph.zero_rhs_columns():
            raise ValueError("every right-hand-side column must be non-zero")

    def _allreduce(self, a, b):
        if self.comm.world > 1 and b > a:
            self.comm.allreduce_(self.ph.red[a:b])

    def step(self) -> int:
        """One mBCG iteration; returns the active-column count after the freeze."""
        it = self.iterations + 1
        if it > self.max_iters:
            raise RuntimeError("mBCG iteration cap exceeded")
        t, k, ph = self.t, self.k, self.ph
        if self.f64:
            P_full = ph.P
            if self.comm.world > 1:
                self.P64_loc[: self.n].copy_(ph.P)
                P_full = self.comm.allgather_rows(self.P64_loc, self.P64_full)
            if self.kv_events is not None:
                self.kv_events[0].record()
            self.mvm.kv.apply64(P_full, t, self.Q)
            if self.kv_events is not None:
                self.kv_events[1].record()
            Q, qf64 = self.Q, True
        elif self.fused:
            if self.comm.world > 1:
                self.comm.allgather_rows(ph.P32, self.P32_full)
            if self.kv_events is not None:
                self.kv_events[0].record()
            self.mvm.kv.apply32(self.P32_full, t, self.Q)
            if self.kv_events is not None:
                self.kv_events[1].record()
            Q, qf64 = self.Q, False
        else:
            Q, qf64 = _apply_user_operator(self.mvm, ph.P, ph.active()), True
        ph.pv(Q, qf64)
        self._allreduce(0, t)
        ph.update(Q, qf64, it)
        self._allreduce(t, 2 * t + (k * t if self.precond is not None else 0))
        ph.precond(it, self.tol)
        self._allreduce(2 * t + k * t, 3 * t + k * t)
        self.iterations = it
        n_active, bad_col, bad_it = ph.status()
        if bad_col < t:
            raise NumericError(f"operator is not positive definite: p^T A p <= 0 for column "
                               f"{bad_col} at iteration {bad_it}")
        if n_active:
            ph.direction(it)
        return n_active

    def run(self) -> "DeviceSolve":
        if self._c_loop_ok():
            return self._run_c_loop()
        while self.iterations < self.max_iters:
            if self.step() == 0:
                break
        return self.finish()

    def _c_loop_ok(self) -> bool:
        """Single device, fused fp32 operator over this state's own rows:
        the whole iteration loop runs in the library (gp_mbcg_solve_kv)."""
        kv = getattr(self.mvm, "kv", None)
        return (self.comm.world == 1 and self.fused and not self.f64 and isinstance(self.ph, CudaPhases)
                and self.kv_events is None and isinstance(kv, _ops.FusedKernelOperator)
                and kv.n_rows == self.n and kv.n_cols == self.n)

    def _run_c_loop(self) -> "DeviceSolve":
        kv, ph, t = self.mvm.kv, self.ph, self.t
        lib = _lib.lib()
        nbytes = lib.gp_kv_workspace_bytes(kv.desc, t)
        ws = _ops.workspace().bytes("kv", nbytes) if nbytes else None
        its = _lib.C.c_int32(0)
        _lib.check(lib.gp_mbcg_solve_kv(ph.sp, _lib.C.byref(kv.desc), _lib.ptr(self.Q), self.Q.stride(0),
                                        _lib.ptr(ws) if ws is not None else 0, int(nbytes), float(self.tol),
                                        _lib.C.byref(its), _lib.stream_handle()), "gp_mbcg_solve_kv")
        self.iterations = int(its.value)
        return self.finish()

    def finish(self) -> "DeviceSolve":
        t, its, tol = self.t, self.iterations, self.tol
        H, rel, conv = self.ph.history(its)
        alphas, betas = [], []
        for j in range(t):
            hit = np.flatnonzero(H[2, :, j] <= tol)
            m = int(hit[0]) + 1 if conv[j] and hit.size else its
            alphas.append([float(x) for x in H[0, :m, j]])
            betas.append([float(x) for x in H[1, :(m - 1 if conv[j] else its), j]])
        return DeviceSolve(self.U, rel, its, alphas, betas, conv, H[2].copy())


def mbcg_device(mvm, B, tol: float, max_iters: int = 1000,
                precond: PreconditionerCache | None = None, comm=None,
                row_offset: int = 0) -> DeviceSolve:
    """Device-resident mBCG on this device's rows of B (n_local x t, fp64)."""
    return MbcgRun(mvm, B, tol, max_iters, precond, comm, row_offset).run()


def _apply_user_operator(mvm, P, active_dev):
    """Apply a user callable to the active columns of P (fp64)."""
    T = D.torch()
    active = D.to_host(active_dev).astype(bool)
    cols = np.flatnonzero(active)
    Q = T.zeros_like(P)
    if cols.size == 0:
        return Q
    idx = T.from_numpy(cols).to(P.device)
    Pa = P.index_select(1, idx)
    try:
        res = mvm(Pa)
    except TypeError:
        res = None
    if res is None or not D.is_tensor(res):
        res = mvm(D.to_host(Pa)) if res is None else res
        res = D.to_device(np.asarray(res, dtype=np.float64))
    res = res.to(T.float64)
    if res.dim() == 1:
        res = res[:, None]
    Q.index_copy_(1, idx, res)
    return Q


def mbcg_solve(mvm, request: SolveRequest) -> SolveReport:
    """Run batched PCG until every column meets the tolerance or the cap
    (cg.py:84-164)."""
    B = D.to_device(request.rhs)
    if B.dim() == 1:
        B = B[:, None]
    sol = mbcg_device(mvm, B, request.tolerance, request.max_iters, request.preconditioner)
    U = sol.U
    return SolveReport(solutions=D.to_host(U), final_relative_residuals=sol.rel,
                       iterations=sol.iterations, tridiagonals=sol.tridiagonals(),
                       converged=sol.converged,
                       residual_history=sol.history if sol.iterations else np.zeros((0, U.shape[1])),
                       solutions_device=U)


def slq_logdet(report, preconditioner: PreconditionerCache | None = None, columns=None,
               n_total: int | None = None) -> float:
    """n * mean_j sum_m (V_0m)^2 log(lambda_m) (+ logdet P) over probe
    columns (cg.py:182-218; the weight is n, as in the reference code).
    `n_total` overrides n for a row-sharded solve (the report holds this
    rank's rows only)."""
    tris = report.tridiagonals if not isinstance(report, DeviceSolve) else report.tridiagonals()
    cols = list(range(len(tris)) if columns is None else columns)
    if not cols:
        raise ValueError("at least one probe column is required")
    n = (report.solutions.shape[0] if isinstance(report, SolveReport) else report.U.shape[0])
    if n_total is not None:
        n = int(n_total)
    # the small eigenproblems of equal order in one batched LAPACK call
    # (the per-column terms are then summed in column order, as before)
    terms = {}
    by_order = {}
    for j in cols:
        if tris[j].order == 0:
            raise NumericError(f"column {j} has an empty recurrence")
        by_order.setdefault(tris[j].order, []).append(j)
    for m, js in by_order.items():
        if m == 1:
            for j in js:
                terms[j] = (tris[j].diag.copy(), np.ones(1))
            continue
        A = np.zeros((len(js), m, m))
        idx = np.arange(m)
        for g, j in enumerate(js):
            A[g, idx, idx] = tris[j].diag
            A[g, idx[1:], idx[:-1]] = tris[j].offdiag
        lam, vecs = np.linalg.eigh(A)   # lower triangle
        for g, j in enumerate(js):
            terms[j] = (lam[g], vecs[g, 0, :] ** 2)
    total = 0.0
    for j in cols:
        lam, w = terms[j]
        if np.any(lam <= 0):
            raise NumericError(f"tridiagonal for column {j} has a non-positive eigenvalue; "
                               "the operator is not positive definite or the recurrence broke down")
        total += float(w @ np.log(lam))
    est = n * total / len(cols)
    if preconditioner is not None:
        est += preconditioner.logdet
    return est
