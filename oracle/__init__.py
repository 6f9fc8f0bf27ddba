"""CPU oracle for the exact-GP BBMM hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy/scipy float64, the algorithm of the
reference package `blockgp` 0.1.0 (`/root/reference/pkg/src/blockgp`) for the
hot path named in BASELINE.json: K̂(X,X)·V, mBCG with Lanczos coefficients,
SLQ log-determinant, rank-k pivoted-Cholesky preconditioner, MLL + gradients,
prediction cache / predictive mean / predictive variance.

Rules:
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
    `--impl reference` leg may import this package, and only as the checker
    or the timed CPU baseline — never as the product path.
  * Parity is pinned: `tests/test_oracle_golden.py` checks this restatement
    against golden vectors produced by running the reference itself
    (`tests/golden/make_golden.py`, committed with its output).
"""

from .blockgp_oracle import *  # noqa: F401,F403
