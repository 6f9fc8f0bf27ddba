"""Row-sharded multi-GPU execution (one process per GPU, torch.distributed).

The reference's only parallelism is row partitioning of K̂ (partition.py:
155-183): partition outputs are disjoint and need no
reduction. Here rank r owns the contiguous rows [r*m, min(n, (r+1)*m)),
m = ceil(n / world), of K̂ and of every CG block; X is replicated (O(nd)
per GPU, as in the paper). Per mBCG iteration the exchange is exactly:
  * all-gather of the fp32 search directions P (4 n t bytes in total),
  * reduce-scatter of the symmetric kernel's int64 fixed-point partial sums
    (8 n t bytes in, each rank keeps the slice of its own rows),
  * all-reduce of the fp64 reduction payload [p^T v | ||r||^2 | L^T r | r^T z]
    (3t + kt scalars) in three phases.
The rank-k pivoted-Cholesky factor is built redundantly on every rank (no
communication, identical pivots everywhere); each rank applies Woodbury on
its rows. Gradients and predictive means reduce 1+n_l or m scalars.
"""

from __future__ import annotations

import math


class TorchComm:
    """Collectives over a torch.distributed process group (NCCL on B200,
    gloo in the CPU tests). Rank r owns rows [row0, row1) =
    [r m, min(n, (r + 1) m)) with m = ceil(n / world) rounded up to `align`
    rows (128 = one symmetric-kernel row block, so a rank's rows are one
    contiguous slice of the fixed-point accumulator and the int64 sums can be
    reduce-scattered; align 1 when n is too small for that, < 128 x world).
    Every collective's payload is counted in `bytes` (per kind) so callers can
    report the measured exchange per iteration."""

    def __init__(self, n_total: int, group=None, align: int | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n_total = n_total
        if align is None:
            align = 128 if n_total >= 128 * self.world else 1
        self.align = int(align)
        m = math.ceil(n_total / self.world)
        self.rows_per_rank = (m + self.align - 1) // self.align * self.align
        self.row0 = min(n_total, self.rank * self.rows_per_rank)
        self.row1 = min(n_total, self.row0 + self.rows_per_rank)
        self.bytes = {"all_gather": 0, "all_reduce": 0, "reduce_scatter": 0}

    @property
    def n_local(self) -> int:
        return self.row1 - self.row0

    @property
    def backend(self) -> str:
        return self.dist.get_backend(self.group)

    def allreduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        self.bytes["all_reduce"] += t.numel() * t.element_size()
        return t

    def allgather_rows(self, local, full):
        """full[r*m:(r+1)*m] = local of rank r (local has m rows, zero padded)."""
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(full, local, group=self.group)
        else:  # gloo (CPU tests)
            parts = list(full.chunk(self.world, dim=0))
            self.dist.all_gather(parts, local.contiguous(), group=self.group)
        self.bytes["all_gather"] += full.numel() * full.element_size()
        return full

    def reduce_scatter_(self, out, full):
        """out (length L) = sum over ranks of full[rank L : (rank + 1) L]
        (full has world x L elements): each rank receives the summed slice of
        its own rows."""
        self.dist.reduce_scatter_tensor(out, full, group=self.group)
        self.bytes["reduce_scatter"] += full.numel() * full.element_size()
        return out

    def reset_bytes(self):
        for k in self.bytes:
            self.bytes[k] = 0


_default = {}


def active_comm(n_total: int):
    """The TorchComm the reference-API entry points shard over when they run
    under torch.distributed with more than one rank (torchrun, one process
    per GPU), else None: mll_value_and_grad, build_cache, predict_mean and
    predict_variance keep their signatures and become multi-GPU."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return None
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() < 2:
        return None
    key = (n_total, dist.get_world_size(), dist.get_rank())
    comm = _default.get(key)
    if comm is None:
        comm = _default[key] = TorchComm(n_total)
    return comm


def shard_bounds(n: int, world: int, rank: int):
    m = math.ceil(n / world)
    r0 = min(n, rank * m)
    return r0, min(n, r0 + m)
