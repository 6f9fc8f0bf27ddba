"""Symmetric kernel vs oracle on one case (diagnostic): python scripts/sym_small.py N D FAM T"""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402
from scripts.sym_check import op_for, run, colrel  # noqa: E402

n, d, fam, t = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
rng = np.random.default_rng(0)
X = rng.standard_normal((n, d))
V = rng.standard_normal((n, t))
ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
m = gp.KernelModel(fam, 1.3, ls, 0.2)
ref = O.kernel_mvm(O.make_hp(fam, 1.3, ls, 0.2), X, V)
got = run(op_for(m, X, 3), V)
err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
bad = np.nonzero(err > 1e-4)[0]
print(f"n={n} d={d} {fam} t={t}: colrel {colrel(got, ref):.2e}; bad rows {len(bad)}: {bad[:20]}")
if len(bad):
    # which 64-column tiles' contributions explain the error of the first bad row tile?
    K = O.kernel_rows(O.make_hp(fam, 1.3, ls, 0.2), X, 0, n)
    r0 = (bad[0] // 128) * 128
    rows = slice(r0, min(n, r0 + 128))
    diff = got[rows] - ref[rows]
    for tt in range((n + 63) // 64):
        cols = slice(64 * tt, min(n, 64 * tt + 64))
        part = K[rows, cols] @ V[cols]
        for coef in (1, -1, 2):
            if np.allclose(diff, coef * part, rtol=1e-3, atol=1e-3 * np.abs(part).max()):
                print(f"  rows {r0}..: error == {coef} x tile {tt}")
    print("  diff norm", np.linalg.norm(diff), "row-tile ref norm", np.linalg.norm(ref[rows]))
