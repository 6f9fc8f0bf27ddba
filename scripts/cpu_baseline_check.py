"""Validate bench.py's CPU reference arm (the oracle port) against the real
reference, in the build container (the reference cannot travel to the GPU
box): time blockgp's own partitioned_mvm(training_mvm_oracle(model)) and the
port bench.py times, on the same 1,024 rows x n columns of K̂·V at the bench
workload M1e6, both with all host cores (WorkerPool(workers=cores) inside
threadpool_limits(1), the reference's bench protocol, experiment.py:384-405).

    python scripts/cpu_baseline_check.py > profiles/r02_cpu_baseline_check.json
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import blockgp  # noqa: E402  the reference
from blockgp import kernels as rk  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

import bench  # noqa: E402
from paper_1903_08114_b200 import synthetic as syn  # noqa: E402


def main(rows=1024, reps=2):
    w = syn.WORKLOADS["M1e6"]
    X = syn.whitened_inputs(w.n, w.d, 0)
    V = syn.rhs_block(w.n, bench.T_RHS, 2)
    model = blockgp.KernelModel(w.family, 1.0, w.lengthscales(), 0.1)
    cores = len(os.sched_getaffinity(0))
    rpp = 8
    plan = blockgp.PartitionPlan(n=w.n, rows_per_partition=rpp,
                                 ranges=tuple((s, min(s + rpp, rows)) for s in range(0, rows, rpp)))
    pool = blockgp.WorkerPool(workers=cores)
    oracle = rk.training_mvm_oracle(model)
    ref_t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        with threadpool_limits(1):
            out_ref = blockgp.partitioned_mvm(oracle, X, V, plan, pool)
        ref_t.append(time.perf_counter() - t0)
    import oracle as O
    hp = O.make_hp(w.family, 1.0, w.lengthscales(), 0.1)
    port_t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out_port = O.partitioned_kernel_mvm(lambda Xa, s, e: O.kernel_block(hp, Xa[s:e], X, add_noise=False),
                                            X[:rows], V, O.partition_ranges(rows, rpp), workers=cores)
        port_t.append(time.perf_counter() - t0)
    # same arithmetic (the port omits the sigma^2 diagonal, added in the CG update)
    diff = out_ref[:rows] - (out_port + 0.1 * V[:rows])
    rel = float(np.linalg.norm(diff) / np.linalg.norm(out_ref[:rows]))
    res = {"workload": "M1e6 (n=1e6, d=11, matern32 ARD, t=11)", "rows": rows, "cores": cores,
           "cpu": platform.processor() or platform.machine(),
           "reference_s": min(ref_t), "port_s": min(port_t), "port_over_reference": min(ref_t) / min(port_t),
           "reference_entries_per_s": rows * w.n / min(ref_t), "port_entries_per_s": rows * w.n / min(port_t),
           "relative_difference": rel, "reps": reps,
           "note": "reference = blockgp.partitioned_mvm(training_mvm_oracle) on a PartitionPlan whose ranges "
                   "cover the first `rows` rows (its own code path, unmodified); port = oracle."
                   "partitioned_kernel_mvm as in bench.py's cpu_baseline leg"}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
