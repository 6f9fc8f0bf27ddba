"""Thin tensor-level wrappers over the C-ABI (all work runs in libgpbbmm)."""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _lib


def _T():
    return D.torch()


def _st():
    return _lib.stream_handle()


class Workspace:
    """Grow-only scratch buffers (caller-owned workspace for the C-ABI)."""

    def __init__(self):
        self._bufs = {}

    def bytes(self, name: str, nbytes: int):
        T = _T()
        nbytes = max(int(nbytes), 8)
        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = T.empty(nbytes, dtype=T.uint8, device=D.device())
            self._bufs[name] = b
        return b

    def f64(self, name: str, count: int):
        return self.bytes(name, 8 * max(int(count), 1)).view(_T().float64)


_ws = Workspace()


def workspace() -> Workspace:
    return _ws


class FusedKernelOperator:
    """Rows [r0, r1) of s2*kappa(Xr, Xc) (+ noise I) applied on the fly by
    gp_kv. Xr/Xc are prescaled fp32 point tensors (n x ld32)."""

    def __init__(self, family_code: int, d: int, Xr32, Xc32, outputscale: float, noise: float,
                 diag_offset: int, algo: int = 0, self_offset: int | None = None):
        """self_offset: row i of Xr is column i + self_offset of Xc (training
        operator rows); defaults to diag_offset."""
        if self_offset is None:
            self_offset = diag_offset
        self.desc = _lib.KvDesc(family=family_code, d=d, Xr=_lib.ptr(Xr32), ldr=Xr32.stride(0),
                                n_rows=Xr32.shape[0], Xc=_lib.ptr(Xc32), ldc=Xc32.stride(0),
                                n_cols=Xc32.shape[0], outputscale=float(outputscale),
                                noise=float(noise), diag_offset=int(diag_offset), algo=int(algo),
                                self_offset=int(self_offset))
        self._keep = (Xr32, Xc32)
        self.n_rows = Xr32.shape[0]
        self.n_cols = Xc32.shape[0]

    def apply32(self, V32, t: int, out32=None):
        """out32[:, :t] = K V32[:, :t] (fp32 in, fp32 out)."""
        T = _T()
        if out32 is None:
            out32 = T.empty((self.n_rows, t), dtype=T.float32, device=D.device())
        L = _lib.lib()
        nbytes = L.gp_kv_workspace_bytes(self.desc, t)
        ws = _ws.bytes("kv", nbytes) if nbytes else None
        _lib.check(L.gp_kv(self.desc, _lib.ptr(V32), V32.shape[1], t, _lib.ptr(out32),
                           out32.shape[1], _lib.ptr(ws), int(nbytes), _st()), "gp_kv")
        return out32


class SymShardedKernelOperator:
    """Rows [comm.row0, comm.row1) of the whole square operator
    s2*kappa(X, X) (+ noise I) with the symmetric kernel's work items split
    across the ranks of `comm` (include/gpbbmm.h, gp_kv_sym_partial): each rank
    forms the 64-bit fixed-point partial sums of its items for all n rows, the
    integer sums are reduce-scattered (deterministic; each rank receives the
    slice of its own 128-aligned rows), and each rank finalises its own rows — bitwise equal to the single-device gp_kv result. Every rank
    then evaluates ~n^2/(2 world) kernel entries instead of n^2/world. Falls
    back to the row-tiled kernel (`fallback`) where one device would not use
    the symmetric kernel either (t > 16, or too few points to fill the SMs,
    gp_kv_sym_auto), unless `force` (algo 3) asks for it whenever supported."""

    def __init__(self, family_code: int, d: int, X32_full, outputscale: float, noise: float,
                 diag_offset: int, comm, fallback=None, force: bool = False):
        self.desc = _lib.KvDesc(family=family_code, d=d, Xr=_lib.ptr(X32_full), ldr=X32_full.stride(0),
                                n_rows=X32_full.shape[0], Xc=_lib.ptr(X32_full), ldc=X32_full.stride(0),
                                n_cols=X32_full.shape[0], outputscale=float(outputscale),
                                noise=float(noise), diag_offset=int(diag_offset), algo=0, self_offset=0)
        self._keep = (X32_full,)
        self.comm = comm
        self.row0, self.row1 = comm.row0, comm.row1
        self.n_rows = self.row1 - self.row0
        self.n_cols = X32_full.shape[0]
        self.fallback = fallback
        self.force = bool(force)
        self._acc = None

    def supported(self, t: int) -> bool:
        L = _lib.lib()
        return bool(L.gp_kv_sym_supported(self.desc, t) if self.force else L.gp_kv_sym_auto(self.desc, t))

    def apply32(self, V32_full, t: int, out32=None):
        """out32[:, :t] = rows [row0, row1) of K V32_full[:n, :t]."""
        if not self.supported(t):
            if self.fallback is None:
                raise ValueError(f"symmetric K·V does not take t={t} and no fallback operator was given")
            return self.fallback.apply32(V32_full, t, out32)
        T = _T()
        L = _lib.lib()
        if out32 is None:
            out32 = T.empty((self.n_rows, t), dtype=T.float32, device=D.device())
        comm = self.comm
        ld = int(L.gp_kv_sym_acc_ld(self.desc))
        m = comm.rows_per_rank
        # reduce-scatter when every rank's rows are whole 128-row blocks (the
        # accumulator is row-block major): each rank receives only its own
        # slice (8 m t bytes) instead of the full 8 n t sums
        rs = m % 128 == 0
        full_rows = max(ld, m * comm.world) if rs else ld
        if self._acc is None or self._acc[0].numel() < t * full_rows:
            self._acc = (T.zeros(t * full_rows, dtype=T.int64, device=D.device()),
                         T.zeros(full_rows, dtype=T.int32, device=D.device()),
                         T.empty(t * m, dtype=T.int64, device=D.device()),
                         T.empty(m, dtype=T.int32, device=D.device()))
        acc, bad = self._acc[0][: t * full_rows], self._acc[1][:full_rows]
        nbytes = L.gp_kv_workspace_bytes(self.desc, t)
        ws = _ws.bytes("kv", nbytes)
        _lib.check(L.gp_kv_sym_partial(self.desc, _lib.ptr(V32_full), V32_full.stride(0), t, comm.rank,
                                       comm.world, _lib.ptr(acc), _lib.ptr(bad), _lib.ptr(ws), int(nbytes),
                                       _st()), "gp_kv_sym_partial")
        if rs:
            # rows past ld (padding of the last rank): the kernel writes only
            # t * ld entries, a previous wider call may have left values there
            if full_rows > ld:
                acc[t * ld:].zero_()
                bad[ld:].zero_()
            acc_l, bad_l = self._acc[2][: t * m], self._acc[3][:m]
            comm.reduce_scatter_(acc_l, acc)
            comm.reduce_scatter_(bad_l, bad)
            acc_row0 = self.row0
        else:
            comm.allreduce_(acc)
            comm.allreduce_(bad)
            acc_l, bad_l, acc_row0 = acc, bad, 0
        _lib.check(L.gp_kv_sym_finalize(self.desc, _lib.ptr(V32_full), V32_full.stride(0), t, _lib.ptr(acc_l),
                                        _lib.ptr(bad_l), acc_row0, self.row0, self.row1, _lib.ptr(out32),
                                        out32.stride(0), _lib.ptr(ws), int(nbytes), _st()), "gp_kv_sym_finalize")
        return out32


def training_operator(family_code: int, d: int, X32_full, outputscale: float, noise: float,
                      diag_offset: int, comm=None, algo: int = 0):
    """The K̂ operator a solver on this rank applies: the whole operator on one
    device (gp_kv picks the symmetric kernel itself), or, across ranks, the
    symmetric schedule split by work items with the row-tiled kernel as the
    fallback for shapes it does not take."""
    if comm is None or getattr(comm, "world", 1) == 1:
        return FusedKernelOperator(family_code, d, X32_full, X32_full, outputscale, noise, diag_offset,
                                   algo=algo, self_offset=0)
    r0, r1 = comm.row0, comm.row1
    rows = FusedKernelOperator(family_code, d, X32_full[r0:r1], X32_full, outputscale, noise,
                               diag_offset + r0 if diag_offset >= 0 else -1, algo=algo, self_offset=r0)
    if algo not in (0, 3):
        return rows
    return SymShardedKernelOperator(family_code, d, X32_full, outputscale, noise, diag_offset, comm,
                                    fallback=rows, force=algo == 3)


def kv_f64(family_code: int, d: int, Xr64, Xc64, outputscale: float, noise: float, diag_offset: int, V,
           out=None):
    """fp64 fused K(Xr, Xc)·V (+ noise V on the diagonal when diag_offset >= 0)
    on gp_kv_f64 — the reference-precision operator (float64 end to end).
    Xr64 / Xc64 are prescaled fp64 points. Returns (out, first non-finite
    row or None)."""
    T = _T()
    V = V.to(T.float64)
    if V.dim() == 1:
        V = V[:, None]
    V = V.contiguous()
    nr, nc, t = Xr64.shape[0], Xc64.shape[0], V.shape[1]
    if out is None:
        out = T.empty((nr, t), dtype=T.float64, device=D.device())
    L = _lib.lib()
    nbytes = L.gp_kv_f64_workspace_bytes(nr, nc, t)
    ws = _ws.bytes("kv_f64", nbytes) if nbytes else None
    bad = T.full((1,), nr, dtype=T.int32, device=D.device())
    _lib.check(L.gp_kv_f64(family_code, d, _lib.ptr(Xr64), Xr64.stride(0), nr, _lib.ptr(Xc64), Xc64.stride(0),
                           nc, float(outputscale), float(noise), int(diag_offset), _lib.ptr(V), V.stride(0), t,
                           _lib.ptr(out), out.stride(0), _lib.ptr(bad), _lib.ptr(ws), int(nbytes), _st()),
               "gp_kv_f64")
    first = int(bad.item())
    return out, (None if first >= nr else first)


class Kv64Operator:
    """Rows of s2*kappa(Xr, Xc) applied in fp64 by gp_kv_f64 (no noise: the
    CG kernels add noise*P): the reference-precision operator an mBCG solve
    uses when CgConfig.precision == "fp64". Xr64/Xc64 are prescaled fp64
    points."""

    def __init__(self, family_code: int, d: int, Xr64, Xc64, outputscale: float):
        self.family_code, self.d = family_code, d
        self.Xr64, self.Xc64 = Xr64, Xc64
        self.outputscale = float(outputscale)
        self.n_rows, self.n_cols = Xr64.shape[0], Xc64.shape[0]

    def apply64(self, V64_full, t: int, out64=None):
        out, bad = kv_f64(self.family_code, self.d, self.Xr64, self.Xc64, self.outputscale, 0.0, -1,
                          V64_full[: self.n_cols, :t], out64)
        return out


def coldot(A, B):
    """Per-column sum(A * B) of two (n, t) fp64 tensors -> (t,) fp64."""
    T = _T()
    n, t = A.shape
    out = T.empty(t, dtype=T.float64, device=D.device())
    part = _ws.f64("coldot", (2 * 148 + 8) * t + 1024)
    _lib.check(_lib.lib().gp_coldot(n, t, _lib.ptr(A), A.stride(0), _lib.ptr(B), B.stride(0),
                                    _lib.ptr(out), _lib.ptr(part), part.numel(), _st()), "gp_coldot")
    return out


def lt_mul(L, V):
    """L^T V for L (n, k), V (n, t) fp64 -> (k, t)."""
    T = _T()
    n, k = L.shape
    t = V.shape[1]
    out = T.empty((k, t), dtype=T.float64, device=D.device())
    part = _ws.f64("ltmul", (2 * 148 + 8) * k * t + 1024)
    _lib.check(_lib.lib().gp_lt_mul(n, k, _lib.ptr(L), L.stride(0), _lib.ptr(V), V.stride(0), t,
                                    _lib.ptr(out), _lib.ptr(part), part.numel(), _st()), "gp_lt_mul")
    return out


def lowrank_mul(L, M, Y=None, alpha=1.0, beta=0.0):
    """Y = beta Y + alpha L M  (L (n,k), M (k,t))."""
    T = _T()
    n, k = L.shape
    t = M.shape[1]
    if Y is None:
        Y = T.empty((n, t), dtype=T.float64, device=D.device())
        beta = 0.0
    M = M.contiguous()
    _lib.check(_lib.lib().gp_lowrank_mul(n, k, _lib.ptr(L), L.stride(0), _lib.ptr(M), M.stride(0), t,
                                         float(alpha), float(beta), _lib.ptr(Y), Y.stride(0), _st()),
               "gp_lowrank_mul")
    return Y


def block_mvm(block, V):
    """(block @ V, first non-finite row or None) for a materialised fp64 block."""
    T = _T()
    nr, nc = block.shape
    t = V.shape[1]
    out = T.empty((nr, t), dtype=T.float64, device=D.device())
    bad = T.full((1,), nr, dtype=T.int32, device=D.device())
    _lib.check(_lib.lib().gp_block_mvm(_lib.ptr(block), nr, nc, block.stride(0), _lib.ptr(V),
                                       V.stride(0), t, _lib.ptr(out), t, _lib.ptr(bad), _st()),
               "gp_block_mvm")
    first = int(bad.item())
    return out, (None if first >= nr else first)


def first_nonfinite_row(A) -> int | None:
    """Index of the first row of a device tensor holding a non-finite value."""
    T = _T()
    bad = ~T.isfinite(A)
    if A.dim() > 1:
        bad = bad.any(dim=1)
    idx = T.nonzero(bad)
    return int(idx[0, 0]) if idx.numel() else None


def np_f64(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64)
