"""Checks of the symmetric K·V kernel (algo 3) against the row-tiled tcgen05
kernel (algo 2) and the fp64 oracle, bitwise reproducibility, and per-launch
timing of both at a given n (run on a B200). Not part of the test suite."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402  (checker only)
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402


def op_for(m, X, algo, noise_diag=True):
    ps = D.points(X)
    Xs32, _ = ps.scaled(m.scale_for(ps.d))
    return _ops.FusedKernelOperator(m.family_code, ps.d, Xs32, Xs32, m.outputscale, m.noise,
                                    0 if noise_diag else -1, algo=algo, self_offset=0)


def colrel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)))


def run(op, V):
    V32 = torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)).cuda()
    return op.apply32(V32, V.shape[1]).double().cpu().numpy()


def small():
    rng = np.random.default_rng(0)
    worst = 0.0
    for n in (1, 5, 64, 127, 128, 129, 191, 256, 700, 3000):
        for d in (1, 3, 11, 14):
            for fam in ("rbf", "matern32"):
                for t in (1, 11, 16):
                    X = rng.standard_normal((n, d))
                    V = rng.standard_normal((n, t))
                    ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
                    m = gp.KernelModel(fam, 1.3, ls, 0.2)
                    ref = O.kernel_mvm(O.make_hp(fam, 1.3, ls, 0.2), X, V)
                    got = run(op_for(m, X, 3), V)
                    e = colrel(got, ref)
                    worst = max(worst, e)
                    if e > 1e-4 or not np.isfinite(e):
                        print(f"FAIL n={n} d={d} {fam} t={t}: colrel {e:.3e}")
    print(f"small cases: worst colrel vs oracle {worst:.2e}")


def large(n, d, fam, reps=3):
    X = syn.whitened_inputs(n, d, 0)
    ls = np.linspace(0.75, 1.5, d)
    m = gp.KernelModel(fam, 1.0, ls, 0.1)
    V = syn.rhs_block(n, 11, 2)
    V32 = torch.from_numpy(V).float().cuda()
    res = {}
    for algo in (2, 3):
        op = op_for(m, X, algo)
        out = op.apply32(V32, 11)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            op.apply32(V32, 11, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[algo] = (out.double().cpu().numpy(), ms)
        ent = n * n / (ms / 1e3)
        print(f"n={n} d={d} {fam} algo={algo}: {ms:.2f} ms/launch, {ent / 1e9:.0f} Gentries/s (n^2)")
    a2, a3 = res[2][0], res[3][0]
    print(f"  colrel(sym, tc) = {colrel(a3, a2):.2e}; speed-up {res[2][1] / res[3][1]:.2f}x")
    again = run(op_for(m, X, 3), V)
    print(f"  bitwise reproducible: {np.array_equal(again, a3)}")
    rows = (n // 3, n // 3 + 64)
    ref = O.kernel_rows(O.make_hp(fam, 1.0, ls, 0.1), X, *rows) @ V
    print(f"  rows {rows}: colrel sym {colrel(a3[rows[0]:rows[1]], ref):.2e}, "
          f"tc {colrel(a2[rows[0]:rows[1]], ref):.2e}")


if __name__ == "__main__":
    small()
    large(65536, 8, "matern32")
    large(278_319, 3, "rbf")
    if "--big" in sys.argv:
        large(1_000_000, 11, "matern32", reps=2)
