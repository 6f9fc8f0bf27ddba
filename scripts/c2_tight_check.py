import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from test_gpu_large_configs import _c2_problem, _c2_mll
from conftest import load_golden
g, w, X, y, m = _c2_problem()
gt = load_golden("c2_tight")
ref = gt["grad_vals"]; keys = [str(k) for k in gt["grad_keys"]]
for prec in ("fp64", "fp32"):
    t0 = time.time()
    r = _c2_mll(m, w, X, y, 0.01, prec)
    got = np.array([r.gradients[k] for k in keys])
    print(prec, "its", r.diagnostics.iterations, "ref", int(gt["iterations"]), "value rel", abs(r.value - float(gt["value"])) / abs(float(gt["value"])),
          "grad", np.abs(got - ref).max() / np.abs(ref).max(), "logdet rel", abs(r.diagnostics.logdet_estimate - float(gt["logdet"])) / abs(float(gt["logdet"])),
          "quad rel", abs(r.diagnostics.quad_term - float(gt["quad"])) / abs(float(gt["quad"])), f"{time.time()-t0:.1f}s")
