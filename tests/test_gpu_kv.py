"""GPU parity of the fused K̂·V path (gp_kv through the C-ABI) against the
reference's golden vectors and the oracle. Tolerance (north_star): relative
1e-4 per column norm for fp32 paths; fp64 paths (dense blocks, user row
oracles) at 1e-12 like the reference's own tests."""

import numpy as np
import pytest

import oracle as O
import paper_1903_08114_b200 as gp
from paper_1903_08114_b200 import kernels, synthetic as syn
from conftest import hp_from, load_golden

pytestmark = pytest.mark.gpu
KV_RTOL = 1e-4


def colrel(got, exp):
    got, exp = np.atleast_2d(got.T).T, np.atleast_2d(exp.T).T
    return np.max(np.linalg.norm(got - exp, axis=0) / np.linalg.norm(exp, axis=0))


def model_of(hp):
    return gp.KernelModel(hp["family"], hp["s2"], hp["ls"], hp["noise"], mean=hp.get("mean", 0.0))


def test_kv_small_goldens():
    g = load_golden("kv_small")
    for c in range(int(g["ncases"])):
        hp = hp_from(g, f"c{c}_")
        m = model_of(hp)
        X, V = g[f"c{c}_X"], g[f"c{c}_V"]
        n = X.shape[0]
        for rows in (1, 7, n):
            got = gp.partitioned_mvm(kernels.training_mvm_oracle(m), X, V,
                                     gp.plan_partitions(n, rows), gp.WorkerPool(workers=2))
            assert colrel(got, g[f"c{c}_KV"]) <= KV_RTOL, (c, rows)
        got = gp.partitioned_mvm(kernels.cross_mvm_oracle(m, X), g[f"c{c}_Xt"], V[:, 0],
                                 gp.plan_partitions(33, 5), gp.WorkerPool())
        assert colrel(got, g[f"c{c}_Kxv"]) <= KV_RTOL, c
        # fp64 dense block path
        blk = kernels.kernel_block(m, X[:7], X[:9])
        np.testing.assert_allclose(blk, g[f"c{c}_block"][:7, :9] - np.where(
            np.eye(7, 9) > 0, hp["noise"], 0.0), rtol=1e-12, atol=1e-13)


def test_bitwise_identical_across_plans_and_pools():
    g = load_golden("kv_small")
    hp = hp_from(g, "c3_")
    m = model_of(hp)
    X, V = g["c3_X"], g["c3_V"]
    res = [gp.partitioned_mvm(kernels.training_mvm_oracle(m), X, V, gp.plan_partitions(120, r),
                              gp.WorkerPool(workers=w)) for r, w in ((13, 1), (13, 2), (120, 3), (1, 1))]
    for r in res[1:]:
        assert np.array_equal(res[0], r)


def test_kernel_rows_and_eval_fp64():
    hp = O.make_hp("matern32", 1.0, [1.0], 0.1)
    m = model_of(hp)
    assert kernels.kernel_eval(m, [0.0], [1.0]) == pytest.approx(0.4833577245965077, rel=1e-14)
    assert kernels.kernel_eval(gp.KernelModel("rbf", 1.0, [1.0], 0.1), [0.0], [1.0]) == \
        pytest.approx(0.6065306597126334, rel=1e-14)
    X = np.random.default_rng(3).uniform(size=(40, 3))
    np.testing.assert_allclose(kernels.kernel_rows(m, X, 5, 9), O.kernel_rows(hp, X, 5, 9),
                               rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(kernels.kernel_block(m, X, X, add_noise=True),
                               O.kernel_block(hp, X, X, add_noise=True), rtol=1e-12, atol=1e-13)
    with pytest.raises(ValueError):
        kernels.kernel_block(m, X[:3], X[:4], add_noise=True)


def test_user_row_oracles():
    """Shipped reference tests on the callable path (test_partition.py:57-128)."""
    def eye_rows(X, a, b):
        out = np.zeros((b - a, X.shape[0]))
        out[np.arange(b - a), np.arange(a, b)] = 1.0
        return out
    v = np.array([1.0, 2.0, 3.0])
    for rows in (1, 2, 3):
        np.testing.assert_array_equal(
            gp.partitioned_mvm(eye_rows, np.zeros((3, 1)), v, gp.plan_partitions(3, rows), gp.WorkerPool()), v)

    def poisoned(X, a, b):
        blk = np.ones((b - a, X.shape[0]))
        if a <= 5 < b:
            blk[5 - a, 0] = np.nan
        return blk
    with pytest.raises(gp.NumericError, match="partition 1"):
        gp.partitioned_mvm(poisoned, np.zeros((10, 1)), np.ones(10), gp.plan_partitions(10, 4), gp.WorkerPool())
    m = gp.KernelModel("rbf", 1.0, [0.4], 0.5)
    X = np.random.default_rng(0).uniform(size=(10, 2))
    with pytest.raises(ValueError):
        gp.partitioned_mvm(kernels.training_mvm_oracle(m), X, np.ones((7, 2)), gp.plan_partitions(10, 4), gp.WorkerPool())
    with pytest.raises(ValueError, match="scratch"):
        gp.partitioned_mvm(kernels.training_mvm_oracle(m), X, np.ones(10), gp.plan_partitions(10, 5),
                           gp.WorkerPool(workers=1, scratch_entries=10))


def test_nonfinite_inputs_name_partition():
    m = gp.KernelModel("rbf", 1.0, [0.4], 0.5)
    X = np.random.default_rng(0).uniform(size=(12, 2))
    X[6, 1] = np.nan  # poisons row 6 AND column 6: the reference fails at partition 0
    with pytest.raises(gp.NumericError, match="partition 0"):
        gp.partitioned_mvm(kernels.training_mvm_oracle(m), X, np.ones(12), gp.plan_partitions(12, 4), gp.WorkerPool())


def _kv_rows(w, X, V, start, rows, algo=0):
    """K̂[start:start+rows, :] V through the C-ABI operator."""
    import torch
    from paper_1903_08114_b200 import _device as D, _ops
    m = gp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    ps = D.points(X)
    Xs32, _ = ps.scaled(m.lengthscales)
    op = _ops.FusedKernelOperator(m.family_code, w.d, Xs32[start:start + rows], Xs32,
                                  m.outputscale, m.noise, start, algo=algo)
    V32 = torch.from_numpy(V).float().cuda()
    return op.apply32(V32, V.shape[1]).double().cpu().numpy()


@pytest.mark.parametrize("key", ["C2", "C3", "C4", "C5", "M1e6"])
def test_row_subsets_large_configs(key):
    """Golden rows of K̂·V produced by the reference at full n."""
    g = load_golden("row_subsets")
    w = syn.WORKLOADS[key]
    X = syn.whitened_inputs(w.n, w.d, 0)
    np.testing.assert_array_equal(np.array([X.sum(), (X * X).sum(), X[17].sum()]), g[f"{key}_X_checksum"])
    V = syn.rhs_block(w.n, 11, 2)
    rows = int(g[f"{key}_rows"])
    for s, exp in zip(g[f"{key}_starts"], g[f"{key}_KV"]):
        got = _kv_rows(w, X, V, int(s), rows)
        assert colrel(got, exp) <= KV_RTOL, (key, s, colrel(got, exp))


@pytest.mark.parametrize("key", ["C2", "C3", "C5", "M1e6"])
def test_symmetric_full_operator_vs_reference_rows(key):
    """The default training operator (symmetric kernel, whole square
    operator in one launch) at full size, checked on the reference's golden
    rows."""
    g = load_golden("row_subsets")
    w = syn.WORKLOADS[key]
    X = syn.whitened_inputs(w.n, w.d, 0)
    V = syn.rhs_block(w.n, 11, 2)
    full = _kv_rows(w, X, V, 0, w.n, algo=3)
    rows = int(g[f"{key}_rows"])
    for s, exp in zip(g[f"{key}_starts"], g[f"{key}_KV"]):
        s = int(s)
        assert colrel(full[s:s + rows], exp) <= KV_RTOL, (key, s, colrel(full[s:s + rows], exp))


def test_row_shards_bitwise_equal_full():
    """Row sharding (the multi-GPU decomposition) reproduces the full product
    bit-for-bit: per-row reduction order depends only on the column count."""
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(w.n, w.d, 0)[:20_000]
    V = syn.rhs_block(20_000, 11, 2)
    full = _kv_rows(w, X, V, 0, 20_000, algo=1)
    for shards in (2, 3, 8):
        b = np.linspace(0, 20_000, shards + 1).astype(int)
        parts = np.vstack([_kv_rows(w, X, V, b[i], b[i + 1] - b[i], algo=1) for i in range(shards)])
        assert np.array_equal(parts, full), shards


# --------------------------------------------------------------------------
# tcgen05 kernel (algo=2) vs the reference goldens / SIMT kernel
# --------------------------------------------------------------------------

def _kv(m, X, V, algo, rows=None, Xc=None):
    import torch
    from paper_1903_08114_b200 import _device as D, _ops
    ps = D.points(X)
    ls = m.scale_for(ps.d)
    Xs32, _ = ps.scaled(ls)
    if Xc is None:
        r0, r1 = rows if rows else (0, ps.n)
        op = _ops.FusedKernelOperator(m.family_code, ps.d, Xs32[r0:r1], Xs32, m.outputscale, m.noise, r0,
                                      algo=algo)
    else:
        cs = D.points(Xc)
        Xc32, _ = cs.scaled(ls)
        op = _ops.FusedKernelOperator(m.family_code, ps.d, Xs32, Xc32, m.outputscale, 0.0, -1, algo=algo)
    V32 = torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)).cuda()
    return op.apply32(V32, V.shape[1]).double().cpu().numpy()


def test_tc_kernel_compiled():
    from paper_1903_08114_b200 import _lib
    assert _lib.lib().gp_has_tcgen05() == 1


def test_tc_small_goldens():
    g = load_golden("kv_small")
    for c in range(int(g["ncases"])):
        hp = hp_from(g, f"c{c}_")
        m = model_of(hp)
        X, V = g[f"c{c}_X"], g[f"c{c}_V"]
        got = _kv(m, X, V, algo=2)
        assert colrel(got, g[f"c{c}_KV"]) <= KV_RTOL, (c, colrel(got, g[f"c{c}_KV"]))
        got = _kv(m, g[f"c{c}_Xt"], V[:, :1], algo=2, Xc=X)
        assert colrel(got[:, 0], g[f"c{c}_Kxv"]) <= KV_RTOL, c


@pytest.mark.parametrize("key", ["C2", "C3", "C4", "C5", "M1e6"])
def test_tc_row_subsets_large_configs(key):
    g = load_golden("row_subsets")
    w = syn.WORKLOADS[key]
    X = syn.whitened_inputs(w.n, w.d, 0)
    V = syn.rhs_block(w.n, 11, 2)
    rows = int(g[f"{key}_rows"])
    for s, exp in zip(g[f"{key}_starts"], g[f"{key}_KV"]):
        got = _kv_rows(w, X, V, int(s), rows, algo=2)
        assert colrel(got, exp) <= KV_RTOL, (key, s, colrel(got, exp))


def test_tc_row_shards_bitwise_equal_full():
    w = syn.WORKLOADS["C5"]
    X = syn.whitened_inputs(w.n, w.d, 0)[:30_000]
    V = syn.rhs_block(30_000, 11, 2)
    full = _kv_rows(w, X, V, 0, 30_000, algo=2)
    simt = _kv_rows(w, X, V, 0, 30_000, algo=1)
    assert colrel(full, simt) <= 1e-5
    for shards in (2, 3, 8):
        b = np.linspace(0, 30_000, shards + 1).astype(int)
        parts = np.vstack([_kv_rows(w, X, V, b[i], b[i + 1] - b[i], algo=2) for i in range(shards)])
        assert np.array_equal(parts, full), shards


@pytest.mark.parametrize("t", [1, 3, 11, 16, 17, 40, 256])
def test_tc_widths_and_families(t):
    """t <= 16: row-tiled tcgen05 kernel; 16 < t <= 256: the wide-RHS kernel
    (variance solves batch 256 test points, predictor.py:135-182)."""
    rng = np.random.default_rng(t)
    for fam in ("rbf", "matern32"):
        for d in (1, 3, 8, 30):
            n = 700
            X = rng.standard_normal((n, d))
            V = rng.standard_normal((n, t))
            ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
            m = gp.KernelModel(fam, 1.3, ls, 0.2)
            ref = O.kernel_mvm(O.make_hp(fam, 1.3, ls, 0.2), X, V)
            got = _kv(m, X, V, algo=2 if t <= 16 else 0)
            assert colrel(got, ref) <= KV_RTOL, (fam, d, t, colrel(got, ref))


def test_wide_rhs_scaled_columns_and_cross_blocks():
    """Wide kernel with columns of very different magnitude (per-column fp16
    scaling) and on cross blocks (test rows x training columns)."""
    rng = np.random.default_rng(7)
    n, d, t = 3000, 8, 100
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, t)) * np.geomspace(1e-6, 1e6, t)
    ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
    m = gp.KernelModel("matern32", 1.1, ls, 0.3)
    hp = O.make_hp("matern32", 1.1, ls, 0.3)
    assert colrel(_kv(m, X, V, algo=0), O.kernel_mvm(hp, X, V)) <= KV_RTOL
    Xt = rng.standard_normal((300, d))
    got = _kv(m, Xt, V, algo=0, Xc=X)
    ref = O.kernel_block(hp, Xt, X) @ V
    assert colrel(got, ref) <= KV_RTOL


def test_symmetric_kernel_matches_row_tiled_and_is_deterministic():
    """algo 3 (each unordered pair once, 64-bit fixed-point accumulation):
    same values as the row-tiled kernel within fp32 round-off, bitwise
    reproducible run to run."""
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(20_000, w.d, 0)
    V = syn.rhs_block(20_000, 11, 2)
    sym = _kv_rows(w, X, V, 0, 20_000, algo=3)
    tc = _kv_rows(w, X, V, 0, 20_000, algo=2)
    assert colrel(sym, tc) <= 1e-5
    assert np.array_equal(sym, _kv_rows(w, X, V, 0, 20_000, algo=3))
    # the default for the whole square operator
    assert np.array_equal(sym, _kv_rows(w, X, V, 0, 20_000, algo=0))


@pytest.mark.parametrize("fam", ["rbf", "matern32"])
def test_symmetric_kernel_edges_vs_oracle(fam):
    """Ragged tile / block edges (n not a multiple of 128 or 512), tiny n,
    d up to the kernel's limit, 1..16 right-hand sides, against the fp64
    oracle."""
    import oracle as O
    import torch
    from paper_1903_08114_b200 import _device as D, _ops
    rng = np.random.default_rng(5)
    for n, d, t in ((1, 3, 1), (5, 1, 16), (129, 14, 11), (700, 11, 16), (2051, 8, 3)):
        X = rng.standard_normal((n, d))
        V = rng.standard_normal((n, t))
        ls = np.linspace(0.75, 1.5, d) * np.sqrt(d)
        m = gp.KernelModel(fam, 1.3, ls, 0.2)
        Xs32, _ = D.points(X).scaled(m.scale_for(d))
        op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, m.outputscale, m.noise, 0, algo=3)
        got = op.apply32(torch.from_numpy(V).float().cuda(), t).double().cpu().numpy()
        ref = O.kernel_mvm(O.make_hp(fam, 1.3, ls, 0.2), X, V)
        assert colrel(got, ref) <= KV_RTOL, (n, d, t, colrel(got, ref))


def test_symmetric_kernel_propagates_nonfinite_inputs():
    """A NaN coordinate poisons its row and column of K̂: the symmetric
    kernel's fixed-point path flags the rows (NaN out), never a finite value."""
    import torch
    from paper_1903_08114_b200 import _device as D, _ops
    rng = np.random.default_rng(3)
    n, d, t = 1000, 6, 11
    X = rng.standard_normal((n, d))
    X[417, 2] = np.nan
    V = rng.standard_normal((n, t))
    m = gp.KernelModel("matern32", 1.0, np.ones(d), 0.1)
    Xs32, _ = D.points(X).scaled(m.scale_for(d))
    op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.1, 0, algo=3)
    out = op.apply32(torch.from_numpy(V).float().cuda(), t).cpu().numpy()
    assert np.isnan(out[417]).all()
    assert not np.isfinite(out).all(axis=1).any(), "a row touching the NaN column came out finite"
