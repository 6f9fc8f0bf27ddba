"""Pin the CPU oracle (oracle/) against golden vectors produced by running the
reference itself (tests/golden/make_golden.py). CPU only."""

import math

import numpy as np
import pytest

import oracle as O
from conftest import hp_from, load_golden


def test_known_answers():
    g = load_golden("known")
    hp_m = O.make_hp("matern32", 1.0, [1.0], 0.1)
    hp_r = O.make_hp("rbf", 1.0, [1.0], 0.1)
    assert O.kernel_block(hp_m, [[0.0]], [[1.0]])[0, 0] == pytest.approx(float(g["matern_at_1"]), rel=1e-15)
    assert float(g["matern_at_1"]) == pytest.approx(0.4833577245965077, rel=1e-15)
    assert O.kernel_block(hp_r, [[0.0]], [[1.0]])[0, 0] == pytest.approx(float(g["rbf_at_1"]), rel=1e-15)
    rep = O.mbcg(lambda V: np.array([[4.0, 1.0], [1.0, 3.0]]) @ V, np.array([1.0, 2.0]), 1e-12)
    np.testing.assert_allclose(rep["solutions"][:, 0], g["cg2_solution"], rtol=1e-14)
    np.testing.assert_allclose(rep["solutions"][:, 0], [1 / 11, 7 / 11], rtol=1e-14)
    assert rep["iterations"] == int(g["cg2_iterations"]) == 2
    two = O.mbcg(lambda V: 2.0 * V, np.random.default_rng(0).standard_normal((3, 1)), 1e-12)
    assert O.slq_logdet(two, 3) == pytest.approx(float(g["slq_2I3"]), rel=1e-14)
    assert float(g["slq_2I3"]) == pytest.approx(3 * math.log(2), rel=1e-14)
    L, piv, res = O.pivoted_cholesky(lambda i: np.diag([4.0, 1.0])[i], [4.0, 1.0], 1)
    np.testing.assert_array_equal(piv, g["pivchol_piv"])
    np.testing.assert_allclose(L, g["pivchol_L"])
    np.testing.assert_allclose(res, g["pivchol_resid"])
    assert O.precond_build(np.zeros((5, 0)), 0.3)["logdet"] == pytest.approx(float(g["precond_k0_logdet"]))
    hp1 = O.make_hp("rbf", 0.5, [1.0], 0.5)
    r1 = O.mll_value_and_grad(hp1, np.zeros((1, 1)), np.array([0.5]), tol=1e-10, probes=1, rank=0)
    assert r1["value"] == pytest.approx(float(g["mll_n1"]), rel=1e-14)


def test_kv_small_cases():
    g = load_golden("kv_small")
    for c in range(int(g["ncases"])):
        hp = hp_from(g, f"c{c}_")
        X, V = g[f"c{c}_X"], g[f"c{c}_V"]
        got = O.kernel_mvm(hp, X, V)
        np.testing.assert_allclose(got, g[f"c{c}_KV"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(O.kernel_block(hp, g[f"c{c}_Xt"], X) @ V[:, 0],
                                   g[f"c{c}_Kxv"], rtol=1e-12, atol=1e-12)
        ranges = O.partition_ranges(X.shape[0], 7)
        part = O.partitioned_kernel_mvm(lambda X_, s, e: O.kernel_rows(hp, X_, s, e), X, V, ranges, workers=3)
        np.testing.assert_allclose(part, g[f"c{c}_KV"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", ["c1_full", "matern_ard", "noprecond", "tight_tol"])
def test_full_pipeline(name):
    g = load_golden(name)
    hp = hp_from(g)
    res = O.mll_value_and_grad(hp, g["X"], g["y"], tol=float(g["tol"]), probes=int(g["probes"]),
                               rank=int(g["rank"]), probe_seed=0)
    np.testing.assert_allclose(res["Z"], g["Z"], rtol=1e-10, atol=1e-12)
    assert res["iterations"] == int(g["iterations"])
    assert res["value"] == pytest.approx(float(g["value"]), rel=1e-9)
    grads = dict(zip([str(k) for k in g["grad_keys"]], g["grad_vals"]))
    scale = max(abs(v) for v in grads.values())
    for k, v in grads.items():
        assert abs(res["gradients"][k] - v) <= 1e-9 * scale, k
    np.testing.assert_allclose(res["report"]["solutions"], g["solutions"], rtol=1e-8, atol=1e-10)
    if "pivots" in g:
        np.testing.assert_array_equal(res["pivots"], g["pivots"])
        assert res["precond"]["logdet"] == pytest.approx(float(g["precond_logdet"]), rel=1e-11)
    if "cache_weights" in g:
        w, rep = O.build_cache(hp, g["X"], g["y"], rank=int(g["rank"]))
        assert rep["iterations"] == int(g["cache_iterations"])
        # fp64 round-off (BLAS summation order) is amplified by CG at tight
        # tolerance; compare against the weight scale
        wscale = np.abs(g["cache_weights"]).max()
        np.testing.assert_allclose(w, g["cache_weights"], rtol=0, atol=1e-6 * wscale)
        mu = O.predict_mean(hp, g["X"], w, g["X_test"])
        np.testing.assert_allclose(mu, g["pred_mean"], rtol=0, atol=1e-6 * np.abs(g["pred_mean"]).max())
        nv = g["pred_var"].shape[0]
        var, _ = O.predict_variance(hp, g["X"], g["X_test"][:nv], rank=int(g["rank"]))
        np.testing.assert_allclose(var, g["pred_var"], rtol=1e-6, atol=1e-9)


def test_row_subsets_inputs_regenerate():
    """The large-config goldens store only seeds + checksums; the synthetic
    generator must reproduce the reference's inputs bit-for-bit."""
    from paper_1903_08114_b200 import synthetic as syn
    g = load_golden("row_subsets")
    for key in ("C2", "C3"):
        w = syn.WORKLOADS[key]
        X = syn.whitened_inputs(w.n, w.d, 0)
        np.testing.assert_array_equal(np.array([X.sum(), (X * X).sum(), X[17].sum()]),
                                      g[f"{key}_X_checksum"])
        hp = O.make_hp(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
        V = syn.rhs_block(w.n, 11, 2)
        rows = int(g[f"{key}_rows"])
        for s, exp in zip(g[f"{key}_starts"], g[f"{key}_KV"]):
            np.testing.assert_allclose(O.kernel_rows(hp, X, s, s + rows) @ V, exp, rtol=1e-11, atol=1e-11)
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(w.n, w.d, 0)
    hp = O.make_hp(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    pc, piv = O.kernel_precond(hp, X, w.rank)
    np.testing.assert_array_equal(piv, g["C2_pivots"])
    assert pc["logdet"] == pytest.approx(float(g["C2_precond_logdet"]), rel=1e-12)


def test_c4_instance_and_gradient_rows_pin_the_oracle():
    """C4 (d = 90) is non-degenerate (off-diagonal K̂·V carries the columns)
    and the oracle's dK/dtheta blocks reproduce the reference's
    grad_row_products (kernels.py:396-410) on the golden rows."""
    from paper_1903_08114_b200 import synthetic as syn
    g = load_golden("row_subsets")
    w = syn.WORKLOADS["C4"]
    X = syn.whitened_inputs(w.n, w.d, 0)
    np.testing.assert_array_equal(np.array([X.sum(), (X * X).sum(), X[17].sum()]), g["C4_X_checksum"])
    hp = O.make_hp(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    V = syn.rhs_block(w.n, 11, 2)
    rows = int(g["C4_rows"])
    s = int(g["C4_starts"][1])
    exp = g["C4_KV"][1]
    np.testing.assert_allclose(O.kernel_rows(hp, X, s, s + rows) @ V, exp, rtol=1e-10, atol=1e-10)
    diag = (hp["s2"] + hp["noise"]) * V[s:s + rows]
    assert (np.linalg.norm(exp - diag, axis=0) / np.linalg.norm(exp, axis=0)).min() >= 0.5
    gg = load_golden("c4_grad")
    start, r = int(gg["start"]), int(gg["rows"])
    R = np.random.default_rng(int(gg["r_seed"])).standard_normal((w.n, int(gg["width"])))
    pids = [str(p) for p in gg["pids"]]
    blocks = O.grad_blocks(hp, X[start:start + 8], X)
    for i in (0, 1, 45, 90):
        np.testing.assert_allclose(blocks[pids[i]] @ R, gg["products"][i][:8], rtol=1e-9,
                                   atol=1e-9 * np.abs(gg["products"][i]).max())


def test_large_pivots_golden_pins_the_oracle():
    """Rank-100 pivots at the bench workload (n = 10^6) from the oracle's
    restatement of precond.py:58-98 equal the reference's."""
    from paper_1903_08114_b200 import synthetic as syn
    g = load_golden("large_pivots")
    w = syn.WORKLOADS["M1e6"]
    X = syn.whitened_inputs(w.n, w.d, 0)
    hp = O.make_hp(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    pc, piv = O.kernel_precond(hp, X, w.rank)
    np.testing.assert_array_equal(piv, g["M1e6_pivots"])
    assert pc["logdet"] == pytest.approx(float(g["M1e6_precond_logdet"]), rel=1e-12)


def test_oracle_split_and_whiten_matches_reference():
    """data.py:163-196 restated (oracle) against the reference's own output."""
    g = load_golden("whiten")
    Xs, ys, tr, va, te, fm, fs, tm, ts = O.split_and_whiten(g["X_raw"], g["y_raw"], int(g["seed"]))
    for a, b in ((tr, g["train_idx"]), (va, g["val_idx"]), (te, g["test_idx"])):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(Xs, g["X"])
    np.testing.assert_array_equal(ys, g["y"])
    np.testing.assert_array_equal(fs, g["feature_std"])
    assert fs[3] == 1.0   # the constant column keeps a unit divisor
    assert tm == float(g["target_mean"]) and ts == float(g["target_std"])
