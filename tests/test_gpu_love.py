"""LOVE predictive-variance cache (paper_1903_08114_b200/love.py): exact at
full rank, a one-sided (over-)estimate at lower rank, against the exact
variances (dense fp64 / the reference-semantics CG path, predictor.py:135-182)."""

import numpy as np
import pytest

import paper_1903_08114_b200 as gp
from paper_1903_08114_b200 import love

pytestmark = pytest.mark.gpu


def _exact_var(m, X, Xt):
    """k** - k*^T K̂^{-1} k* with dense fp64 blocks (Cholesky)."""
    import torch
    from paper_1903_08114_b200 import kernels, _device as D
    K = kernels.kernel_block_device(m, X, X, add_noise=True)
    Ks = kernels.kernel_block_device(m, X, Xt)
    L = torch.linalg.cholesky(K)
    A = torch.cholesky_solve(Ks, L)
    return D.to_host(m.outputscale - (Ks * A).sum(0))


@pytest.mark.parametrize("fam,ard,n", [("rbf", False, 512), ("matern32", True, 700)])
def test_love_full_rank_is_exact(fam, ard, n):
    rng = np.random.default_rng(n)
    d = 4
    X = rng.standard_normal((n, d))
    Xt = rng.standard_normal((60, d)) * 1.3
    ls = np.linspace(0.8, 1.6, d) if ard else np.array([1.1])
    m = gp.KernelModel(fam, 1.4, ls, 0.15)
    cache = love.build_love_cache(m, X, rank=n, block=16, precision="fp64")
    assert cache.rank == n
    v, clamped = love.predict_variance_love(cache, Xt, precision="fp64")
    ref = _exact_var(m, X, Xt)
    np.testing.assert_allclose(v, ref, rtol=0, atol=1e-9 * m.outputscale)
    assert clamped == 0


def test_love_rank_k_overestimates_and_converges():
    """Q T^{-1} Q^T <= K̂^{-1} (Loewner order), so the rank-k variance is an
    upper bound of the exact one; the gap shrinks as the rank grows."""
    rng = np.random.default_rng(3)
    n, d = 4000, 3
    X = rng.standard_normal((n, d))
    Xt = rng.standard_normal((200, d))
    m = gp.KernelModel("rbf", 1.0, np.array([1.0]), 0.1)
    ref = _exact_var(m, X, Xt)
    gaps = []
    for rank in (32, 128, 256):
        cache = love.build_love_cache(m, X, rank=rank, block=16, precision="fp64")
        v, _ = love.predict_variance_love(cache, Xt, precision="fp64")
        assert np.all(v >= ref - 1e-9)
        gaps.append(np.abs(v - ref).max())
    assert gaps[0] > gaps[1] > gaps[2]
    assert gaps[2] <= 2e-2   # measured: profiles/r02_love.md


def test_love_fp32_operator_and_cross_product_agree_with_fp64():
    rng = np.random.default_rng(9)
    n, d = 20_000, 8
    X = rng.standard_normal((n, d))
    Xt = rng.standard_normal((300, d))
    m = gp.KernelModel("matern32", 1.0, np.linspace(0.75, 1.5, d) * 2.0, 0.1)
    c32 = love.build_love_cache(m, X, rank=128, block=16, precision="fp32")
    c64 = love.build_love_cache(m, X, rank=128, block=16, precision="fp64")
    v32, _ = love.predict_variance_love(c32, Xt, precision="fp32")
    v64, _ = love.predict_variance_love(c64, Xt, precision="fp64")
    np.testing.assert_allclose(v32, v64, rtol=0, atol=1e-4)
