"""Run-to-run determinism of the fused K·V kernels and of a full MLL."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, likelihood as LK, synthetic as syn  # noqa: E402


def main():
    w = syn.WORKLOADS["C2"]
    n = w.n
    X = syn.whitened_inputs(n, w.d, 0)
    y = syn.rff_target(X, features=256)
    m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
    ps = D.points(X)
    Xs32, _ = ps.scaled(m.lengthscales)
    V = torch.from_numpy(syn.rhs_block(n, 11, 2)).float().cuda()
    outs = {}
    for algo in (1, 2):
        op = _ops.FusedKernelOperator(m.family_code, w.d, Xs32, Xs32, 1.0, 0.0, -1, algo=algo, self_offset=0)
        res = [op.apply32(V, 11).clone() for _ in range(5)]
        same = all(torch.equal(res[0], r) for r in res[1:])
        diffs = [float((res[0] - r).abs().max()) for r in res[1:]]
        print(f"algo={algo}: 5 runs bitwise equal: {same}  maxdiff={max(diffs):.3e}")
        outs[algo] = res[0].double()
    rel = ((outs[1] - outs[2]).norm(dim=0) / outs[1].norm(dim=0)).max()
    print(f"SIMT vs tcgen05 full K·V colrel: {float(rel):.3e}")
    for i in range(3):
        r = gp.mll_value_and_grad(m, X, y, gp.plan_partitions(n, n), gp.WorkerPool(), LK.CgConfig(), 0)
        print(f"mll run {i}: value={r.value!r} iters={r.diagnostics.iterations} "
              f"g0={r.gradients['outputscale']!r}")


if __name__ == "__main__":
    main()
