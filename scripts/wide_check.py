"""Wide-RHS K·V kernel checks (diagnostic): small cases vs the fp64 oracle,
large case vs the SIMT kernel, and timing."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402
from paper_1903_08114_b200 import _device as D, _ops, synthetic as syn  # noqa: E402


def colrel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)))


def op_for(m, X, algo, rows=None):
    ps = D.points(X)
    Xs32, _ = ps.scaled(m.scale_for(ps.d))
    r0, r1 = rows or (0, ps.n)
    return _ops.FusedKernelOperator(m.family_code, ps.d, Xs32[r0:r1], Xs32, m.outputscale, m.noise, r0, algo=algo)


rng = np.random.default_rng(0)
worst = 0
for n in (50, 700, 3000):
    for d in (3, 11):
        for fam in ("rbf", "matern32"):
            for t in (17, 40, 100, 256):
                X = rng.standard_normal((n, d))
                V = rng.standard_normal((n, t)) * np.geomspace(1e-3, 1e3, t)
                ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
                m = gp.KernelModel(fam, 1.3, ls, 0.2)
                ref = O.kernel_mvm(O.make_hp(fam, 1.3, ls, 0.2), X, V)
                V32 = torch.from_numpy(V).float().cuda()
                got = op_for(m, X, 0).apply32(V32, t).double().cpu().numpy()
                e = colrel(got, ref)
                worst = max(worst, e)
                if e > 1e-4:
                    print(f"FAIL n={n} d={d} {fam} t={t}: {e:.2e}")
print(f"small wide cases: worst colrel {worst:.2e}")
for n, d, fam in ((65536, 8, "matern32"), (278319, 3, "rbf")):
    X = syn.whitened_inputs(n, d, 0)
    m = gp.KernelModel(fam, 1.0, np.linspace(0.75, 1.5, d), 0.1)
    V = np.random.default_rng(1).standard_normal((n, 256))
    V32 = torch.from_numpy(V).float().cuda()
    res = {}
    for algo in (0, 1):
        op = op_for(m, X, algo)
        out = op.apply32(V32, 256)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply32(V32, 256, out)
        e1.record()
        torch.cuda.synchronize()
        res[algo] = (out.double().cpu().numpy(), e0.elapsed_time(e1))
        print(f"n={n} {fam} t=256 algo={algo}: {res[algo][1]:.1f} ms")
    print(f"  colrel(wide, simt) = {colrel(res[0][0], res[1][0]):.2e}; speed-up {res[1][1] / res[0][1]:.1f}x")
