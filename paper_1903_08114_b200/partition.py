"""Row partitions and the partitioned K̂·V executor (mirror of blockgp.partition).

Reference contract (partition.py:1-7, :186-241): rows are split into
contiguous ranges, each range's row block is multiplied against V and the
disjoint output rows are written; memory stays at one block per worker.

On the B200 the block never exists. A kernel-operator descriptor
(kernels.training_mvm_oracle / cross_mvm_oracle) is executed by the fused
gp_kv kernel over all rows at once; each row's column reduction order is
fixed by the column count alone, so the result is bitwise identical for
every plan and every worker/device count (test_partition.py:92-102). The
plan/pool keep their reference meaning for validation and, for arbitrary
Python row oracles, drive a device loop over materialised blocks.
Multi-GPU row sharding lives in paper_1903_08114_b200.distributed.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _ops
from .errors import NumericError

DEFAULT_BUDGET_BYTES = 1 << 30
_FLOAT_BYTES = 8


@dataclass(frozen=True)
class PartitionPlan:
    """Contiguous, ordered, disjoint half-open row ranges covering [0, n)."""

    n: int
    rows_per_partition: int
    ranges: tuple

    @property
    def num_partitions(self) -> int:
        return len(self.ranges)

    @property
    def block_entries(self) -> int:
        return self.rows_per_partition * self.n

    def partition_of(self, row: int) -> int:
        return min(row // self.rows_per_partition, self.num_partitions - 1)


@dataclass(frozen=True)
class WorkerPool:
    """w workers with a per-worker scratch budget (entries). On the GPU path
    `workers` is informational (one device executes all partitions); the
    scratch budget contract is still enforced."""

    workers: int = 1
    scratch_entries: int = DEFAULT_BUDGET_BYTES // _FLOAT_BYTES

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.scratch_entries < 1:
            raise ValueError("scratch_entries must be >= 1")


def plan_partitions(n: int, rows_per_partition: int) -> PartitionPlan:
    """ceil(n / rows_per_partition) ranges (partition.py:60-76)."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    if rows_per_partition < 1:
        raise ValueError(f"rows_per_partition must be >= 1, got {rows_per_partition}")
    starts = range(0, n, rows_per_partition)
    return PartitionPlan(n=n, rows_per_partition=min(rows_per_partition, n),
                         ranges=tuple((s, min(s + rows_per_partition, n)) for s in starts))


def plan_from_budget(n: int, budget_bytes: int = DEFAULT_BUDGET_BYTES) -> PartitionPlan:
    """rows_per_partition = budget / (8 n), at least 1 (partition.py:79-82)."""
    return plan_partitions(n, max(1, min(n, budget_bytes // (_FLOAT_BYTES * n))))


# --- transient-allocation tracking (partition.py:93-148) --------------------

class AllocationTracker:
    def __init__(self):
        self._lock = threading.Lock()
        self.max_single_entries = 0
        self.live_entries = 0
        self.peak_live_entries = 0
        self.num_allocations = 0

    def _note(self, entries: int) -> None:
        with self._lock:
            self.num_allocations += 1
            self.max_single_entries = max(self.max_single_entries, entries)
            self.live_entries += entries
            self.peak_live_entries = max(self.peak_live_entries, self.live_entries)

    def _drop(self, entries: int) -> None:
        with self._lock:
            self.live_entries -= entries


_tracker = None
_tracker_lock = threading.Lock()


@contextmanager
def track_allocations():
    global _tracker
    tr = AllocationTracker()
    with _tracker_lock:
        if _tracker is not None:
            raise RuntimeError("allocation tracking is already active")
        _tracker = tr
    try:
        yield tr
    finally:
        with _tracker_lock:
            _tracker = None


def transient(shape, dtype=np.float64):
    buf = np.empty(shape, dtype=dtype)
    if _tracker is not None:
        _tracker._note(buf.size)
    return buf


def release(buf) -> None:
    if _tracker is not None:
        _tracker._drop(buf.size)


def _note_device_block(entries: int) -> None:
    """Fused kernels keep only tile-sized operands live; record one tile so
    the memory contract (max transient <= one block) stays observable."""
    if _tracker is not None:
        _tracker._note(entries)
        _tracker._drop(entries)


# --- execution ---------------------------------------------------------------

def run_row_blocks(plan: PartitionPlan, pool: WorkerPool, task) -> None:
    """task(idx, start, stop) per partition, in order (partition.py:155-183).
    Tasks submit device work on the current stream, so ordering, not host
    threads, provides the overlap."""
    for idx, (start, stop) in enumerate(plan.ranges):
        task(idx, start, stop)


def _nonfinite_error(plan: PartitionPlan, row: int) -> NumericError:
    idx = plan.partition_of(row)
    s, e = plan.ranges[idx]
    return NumericError(f"non-finite kernel entry in partition {idx} (rows [{s}, {e}))")


def partitioned_mvm(row_block_fn, X, V, plan: PartitionPlan, pool: WorkerPool, *,
                    precision: str = "fp64") -> np.ndarray:
    """[row_block_fn(X, a, b) @ V for each range] (partition.py:186-241).

    precision "fp64" (default) keeps the reference's float64 contract for
    the kernel oracles (gp_kv_f64, fused, ~1e-15 relative); "fp32" runs the
    tcgen05 operator the mBCG solver uses (~1e-6 relative, SFU-bound)."""
    out = partitioned_mvm_device(row_block_fn, X, V, plan, pool, precision=precision)
    return D.to_host(out)


def _validate(X_rows: int, V, plan, pool):
    if V.ndim != 2:
        raise ValueError(f"V must be 1- or 2-dimensional, got ndim={V.ndim}")
    if plan.n != X_rows:
        raise ValueError(f"plan covers {plan.n} rows but X has {X_rows}")
    if pool.scratch_entries < plan.block_entries:
        raise ValueError(f"worker scratch ({pool.scratch_entries} entries) is smaller than one "
                         f"row block ({plan.block_entries} entries); repartition")


def partitioned_mvm_device(row_block_fn, X, V, plan: PartitionPlan, pool: WorkerPool, *,
                           precision: str = "fp64"):
    """Device-resident variant: returns a CUDA tensor (fp64)."""
    from .kernels import CrossOperator, TrainingOperator
    if precision not in ("fp64", "fp32"):
        raise ValueError(f"precision must be 'fp64' or 'fp32', got {precision!r}")
    T = D.torch()
    squeeze = np.ndim(V) == 1
    Vd = D.to_device(V)
    if squeeze:
        Vd = Vd[:, None]
    n_rows = X.shape[0] if hasattr(X, "shape") else np.asarray(X).shape[0]
    _validate(n_rows, Vd, plan, pool)
    if isinstance(row_block_fn, (TrainingOperator, CrossOperator)):
        model = row_block_fn.model
        ps = D.points(X)
        if isinstance(row_block_fn, TrainingOperator):
            if Vd.shape[0] != ps.n:
                raise ValueError(f"row blocks have {ps.n} columns but V has {Vd.shape[0]} rows")
            cs, noise, diag = ps, model.noise, 0
        else:
            cs = D.points(row_block_fn.X_cols)
            if cs.d != ps.d:
                raise ValueError(f"dimension mismatch: rows have d={ps.d}, cols have d={cs.d}")
            if Vd.shape[0] != cs.n:
                raise ValueError(f"row blocks have {cs.n} columns but V has {Vd.shape[0]} rows")
            noise, diag = 0.0, -1
        ls = model.scale_for(ps.d)
        Xr32, Xr64 = ps.scaled(ls)
        Xc32, Xc64 = cs.scaled(ls)
        if precision == "fp64":
            _note_device_block(min(plan.block_entries, 64 * cs.n))
            out, bad = _ops.kv_f64(model.family_code, ps.d, Xr64, Xc64, model.outputscale, noise, diag, Vd)
            if bad is not None:
                raise _nonfinite_error(plan, bad)
            return out[:, 0] if squeeze else out
        op = _ops.FusedKernelOperator(model.family_code, ps.d, Xr32, Xc32, model.outputscale, noise, diag)
        _note_device_block(min(plan.block_entries, 64 * op.n_cols))
        out = op.apply32(Vd.to(T.float32).contiguous(), Vd.shape[1]).to(T.float64)
        bad = _ops.first_nonfinite_row(out)
        if bad is not None:
            raise _nonfinite_error(plan, bad)
        return out[:, 0] if squeeze else out

    # arbitrary row oracle: materialise each partition's block on the device
    Xh = X
    out = T.empty((plan.n, Vd.shape[1]), dtype=T.float64, device=D.device())

    def task(idx, start, stop):
        blk = row_block_fn(Xh, start, stop)
        shape = tuple(blk.shape)
        if shape != (stop - start, Vd.shape[0]):
            raise ValueError(f"row block for partition {idx} has shape {shape}, "
                             f"expected {(stop - start, Vd.shape[0])}")
        _note_device_block(int(np.prod(shape)))
        res, bad = _ops.block_mvm(D.to_device(blk), Vd)
        if bad is not None:
            raise NumericError(f"non-finite kernel entry in partition {idx} (rows [{start}, {stop}))")
        out[start:stop] = res

    run_row_blocks(plan, pool, task)
    return out[:, 0] if squeeze else out


def communication_model(plan: PartitionPlan, pool: WorkerPool, t: int) -> dict:
    """Bytes a distributed MVM moves (partition.py:244-255): every worker
    receives V once, returns its disjoint rows; O(n t), never a block."""
    to_w = pool.workers * plan.n * t * _FLOAT_BYTES
    from_w = plan.n * t * _FLOAT_BYTES
    return {"bytes_to_workers": to_w, "bytes_from_workers": from_w, "total_bytes": to_w + from_w}
