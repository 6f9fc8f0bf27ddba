"""Accuracy of the fp32 tcgen05 K̂·V kernels (row-tiled algo 2, symmetric algo
3, wide t = 40) against the fp64 kernel (gp_kv_f64, pinned to the oracle at
1e-11) across lengthscale regimes, incl. short ones where most kernel values
are small (the fp16 K split's subnormal range). GPU diagnostic."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops  # noqa: E402


def colrel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)))


rng = np.random.default_rng(0)
for fam in ("matern32", "rbf"):
    for n, d, ls in ((20000, 3, 0.02), (20000, 3, 0.1), (20000, 8, 0.5), (20000, 8, 2.0)):
        X = rng.standard_normal((n, d))
        m = gp.KernelModel(fam, 1.0, np.full(d, ls), 0.01)
        ps = D.points(X)
        Xs32, Xs64 = ps.scaled(m.lengthscales)
        res = []
        for t in (11, 40):
            V = rng.standard_normal((n, t))
            ref, _ = _ops.kv_f64(m.family_code, d, Xs64, Xs64, 1.0, 0.0, -1, torch.from_numpy(V).cuda())
            ref = ref.cpu().numpy()
            for algo in ((2, 3) if t <= 16 else (0,)):
                op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.0, -1, algo=algo, self_offset=0)
                got = op.apply32(torch.from_numpy(V.astype(np.float32)).cuda(), t).double().cpu().numpy()
                res.append(f"t={t} algo={algo}: {colrel(got, ref):.2e}")
        print(f"{fam} n={n} d={d} ls={ls}: " + "  ".join(res), flush=True)
