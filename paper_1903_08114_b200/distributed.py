"""Row-sharded multi-GPU execution (one process per GPU, torch.distributed).

The reference's only parallelism is row partitioning of K̂ (partition.py:
155-183): partition outputs are disjoint and need no
reduction. Here rank r owns the contiguous rows [r*m, min(n, (r+1)*m)),
m = ceil(n / world), of K̂ and of every CG block; X is replicated (O(nd)
per GPU, as in the paper). Per mBCG iteration the exchange is exactly:
  * all-gather of the fp32 search directions P (4 n t bytes in total),
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
    gloo in the CPU tests)."""

    def __init__(self, n_total: int, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n_total = n_total
        self.rows_per_rank = math.ceil(n_total / self.world)
        self.row0 = min(n_total, self.rank * self.rows_per_rank)
        self.row1 = min(n_total, self.row0 + self.rows_per_rank)

    @property
    def n_local(self) -> int:
        return self.row1 - self.row0

    def allreduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def allgather_rows(self, local, full):
        """full[r*m:(r+1)*m] = local of rank r (local has m rows, zero padded)."""
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_gather_into_tensor(full, local, group=self.group)
        else:  # gloo (CPU tests)
            parts = list(full.chunk(self.world, dim=0))
            self.dist.all_gather(parts, local.contiguous(), group=self.group)
        return full


def shard_bounds(n: int, world: int, rank: int):
    m = math.ceil(n / world)
    r0 = min(n, rank * m)
    return r0, min(n, r0 + m)
