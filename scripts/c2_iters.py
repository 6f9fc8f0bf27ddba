"""Diagnose the C2 MLL iteration count: the same [y - mu | Z] block and
preconditioner solved with the symmetric fp32 operator (default), the
row-tiled fp32 operator, and the fp64 operator (gp_kv_f64) as a user
callable. Prints iterations, final residuals and the SLQ/quad terms."""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
from paper_1903_08114_b200.cg import FusedOperator, mbcg_device, slq_logdet  # noqa: E402
from paper_1903_08114_b200.likelihood import build_kernel_preconditioner, draw_probes_device  # noqa: E402


def main(key="C2"):
    import torch
    w = syn.WORKLOADS[key]
    X = syn.whitened_inputs(w.n, w.d, 0)
    y = syn.rff_target(X, seed=1)
    m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    ps = D.points(X)
    Xs32, Xs64 = ps.scaled(m.lengthscales)
    pc = build_kernel_preconditioner(m, ps, w.rank)
    Z = draw_probes_device(w.n, 10, 0, pc)
    B = torch.cat([D.to_device(y)[:, None], Z], dim=1).contiguous()
    V = torch.from_numpy(syn.rhs_block(w.n, 11, 2)).cuda()
    ref64, _ = _ops.kv_f64(m.family_code, w.d, Xs64, Xs64, 1.0, 0.0, -1, V)
    for name, algo in (("sym", 3), ("tc", 2)):
        kv = _ops.FusedKernelOperator(m.family_code, w.d, Xs32, Xs32, 1.0, 0.0, -1, algo=algo, self_offset=0)
        got = kv.apply32(V.float().contiguous(), 11).double()
        colrel = ((got - ref64).norm(dim=0) / ref64.norm(dim=0)).max().item()
        t0 = time.perf_counter()
        sol = mbcg_device(FusedOperator(kv, m.noise, w.n), B, 1.0, 1000, pc)
        el = time.perf_counter() - t0
        ld = slq_logdet(sol, pc, columns=range(1, 11))
        print(f"{name}: K·V colrel vs fp64 {colrel:.2e}; iterations {sol.iterations} ({el:.2f}s) "
              f"logdet {ld:.6f} rel {np.array2string(sol.rel, precision=4)}", flush=True)

    def mvm64(P):
        out, _ = _ops.kv_f64(m.family_code, w.d, Xs64, Xs64, 1.0, m.noise, 0, P)
        return out
    t0 = time.perf_counter()
    sol = mbcg_device(mvm64, B, 1.0, 1000, pc)
    el = time.perf_counter() - t0
    ld = slq_logdet(sol, pc, columns=range(1, 11))
    print(f"fp64: iterations {sol.iterations} ({el:.2f}s) logdet {ld:.6f} "
          f"rel {np.array2string(sol.rel, precision=4)}", flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:]))
