"""Diagnostics for the fused K·V kernels (run on a B200): accuracy of the SIMT
and tcgen05 kernels against the fp64 oracle on row samples, and per-launch
device time at the metric size. Not part of the test suite."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402  (checker only)
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402


def kv(m, X, V, algo, rows=None):
    ps = D.points(X)
    Xs32, _ = ps.scaled(m.lengthscales)
    r0, r1 = rows or (0, ps.n)
    op = _ops.FusedKernelOperator(m.family_code, ps.d, Xs32[r0:r1], Xs32, m.outputscale, m.noise, r0,
                                  algo=algo)
    V32 = torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)).cuda()
    return op, V32


def colrel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)))


def accuracy():
    for label, n, d, fam, ls, center in (("C1-like [0,1]^8 rbf l=.4", 8192, 8, "rbf", [0.4], False),
                                         ("C5-like whitened d=11 matern", 65536, 11, "matern32", None, True),
                                         ("C4-like whitened d=90 matern", 32768, 90, "matern32", None, True),
                                         ("C3-like whitened d=3 rbf", 200000, 3, "rbf", [1.0], True)):
        X = syn.whitened_inputs(n, d, 0) if center else np.random.default_rng(0).uniform(size=(n, d))
        ls = np.asarray(ls if ls is not None else np.linspace(0.75, 1.5, d))
        m = gp.KernelModel(fam, 1.0, ls, 0.1)
        V = syn.rhs_block(n, 11, 2)
        rows = (n // 2, n // 2 + 64)
        ref = O.kernel_rows(O.make_hp(fam, 1.0, ls, 0.1), X, *rows) @ V
        for algo in (1, 2):
            op, V32 = kv(m, X, V, algo, rows)
            got = op.apply32(V32, 11).double().cpu().numpy()
            print(f"{label:34s} algo={algo} colrel={colrel(got, ref):.2e}")


def timing(n=1_000_000):
    w = syn.WORKLOADS["M1e6"]
    X = syn.whitened_inputs(n, w.d, 0)
    m = gp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
    V = syn.rhs_block(n, 11, 2)
    for algo in (2,):
        op, V32 = kv(m, X, V, algo)
        out = op.apply32(V32, 11)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            op.apply32(V32, 11, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        ent = n * n / (ms / 1e3)
        print(f"n={n} algo={algo}: {ms:.1f} ms/launch, {ent / 1e9:.0f} Gentries/s, "
              f"{ent * 44 / 1e12:.1f} TFLOP/s (2d+2t), SFU frac {ent / (148 * 16 * 1.965e9 / 2):.3f}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--timing-only" not in sys.argv:
        accuracy()
    timing(int(args[0]) if args else 1_000_000)
