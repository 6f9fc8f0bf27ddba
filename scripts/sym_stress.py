"""Repeat the symmetric kernel on one case and count mismatching runs (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1903_08114_b200 as gp  # noqa: E402
from scripts.sym_check import op_for  # noqa: E402

n, d, fam, reps = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
rng = np.random.default_rng(0)
X = rng.standard_normal((n, d))
V = rng.standard_normal((n, 11))
ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
m = gp.KernelModel(fam, 1.3, ls, 0.2)
ref = O.kernel_mvm(O.make_hp(fam, 1.3, ls, 0.2), X, V)
op = op_for(m, X, 3)
V32 = torch.from_numpy(V).float().cuda()
nbad = 0
badrows = set()
for r in range(reps):
    got = op.apply32(V32, 11).double().cpu().numpy()
    err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    b = np.nonzero(err > 1e-4)[0]
    if len(b):
        nbad += 1
        badrows.update((b // 64).tolist())
print(f"n={n} d={d} {fam}: {nbad}/{reps} runs wrong; bad 64-row blocks {sorted(badrows)[:20]}")
