"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side logic (plans, transforms, persistence, errors)
matches the reference contract; the product path refuses to run without a
GPU (no CPU fallback)."""

import os
import re

import numpy as np
import pytest

import paper_1903_08114_b200 as gp
from paper_1903_08114_b200 import _lib, kernels, partition, predictor
from conftest import REPO, cuda_ok


def _header_symbols():
    txt = open(os.path.join(REPO, "include", "gpbbmm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gp_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    so = _lib.load_library()
    declared = _header_symbols()
    assert declared, "no symbols parsed from include/gpbbmm.h"
    assert set(declared) == set(_lib.EXPORTED), set(declared) ^ set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(so, name), name
    assert so.gp_version() >= 1
    # query entry points are host-only and safe without a device
    assert so.gp_pivchol_workspace_bytes(1000, 10) > 0


def test_library_has_sm100a_code():
    path = _lib.LIB_PATH
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


@pytest.mark.skipif(cuda_ok(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_gpu():
    X = np.random.default_rng(0).uniform(size=(10, 2))
    model = gp.KernelModel("rbf", 1.0, [0.5], 0.1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        gp.partitioned_mvm(kernels.training_mvm_oracle(model), X, np.ones(10),
                           gp.plan_partitions(10, 4), gp.WorkerPool())


class TestPlans:  # mirrors test_partition.py:17-53 of the reference
    def test_ceiling_arithmetic(self):
        plan = gp.plan_partitions(10, 3)
        assert plan.ranges == ((0, 3), (3, 6), (6, 9), (9, 10))
        assert plan.num_partitions == 4

    def test_single_partition(self):
        assert gp.plan_partitions(5, 5).ranges == ((0, 5),)

    def test_houseelectric_partition_count(self):
        n = 1_311_539
        assert gp.plan_partitions(n, -(-n // 218)).num_partitions == 218

    def test_cover_disjoint(self):
        for n, rows in [(1, 1), (17, 4), (100, 7), (64, 64), (64, 100)]:
            seen = [i for s, e in gp.plan_partitions(n, rows).ranges for i in range(s, e)]
            assert seen == list(range(n))

    def test_invalid(self):
        with pytest.raises(ValueError):
            gp.plan_partitions(0, 3)
        with pytest.raises(ValueError):
            gp.plan_partitions(10, 0)
        with pytest.raises(ValueError):
            gp.WorkerPool(workers=0)

    def test_budget(self):
        plan = gp.plan_from_budget(10_000, budget_bytes=8 * 10_000 * 250)
        assert plan.rows_per_partition == 250

    def test_partition_of(self):
        plan = gp.plan_partitions(10, 4)
        assert [plan.partition_of(r) for r in range(10)] == [0] * 4 + [1] * 4 + [2] * 2

    def test_communication_model(self):
        plan = gp.plan_partitions(50_000, 1000)
        pool = gp.WorkerPool(workers=4, scratch_entries=plan.block_entries)
        b = partition.communication_model(plan, pool, 8)["total_bytes"]
        assert b == 5 * 50_000 * 8 * 8 and b * 100 < 50_000 ** 2 * 8


class TestModel:
    def test_validation(self):
        with pytest.raises(ValueError):
            gp.KernelModel("cubic", 1.0, [1.0], 0.1)
        with pytest.raises(ValueError):
            gp.KernelModel("rbf", -1.0, [1.0], 0.1)
        with pytest.raises(ValueError):
            gp.KernelModel("rbf", 1.0, [0.0], 0.1)
        with pytest.raises(ValueError):
            gp.KernelModel("rbf", 1.0, [1.0], 0.1, noise_floor=0.2)
        with pytest.raises(ValueError):
            gp.KernelModel("rbf", 1.0, [1.0, 2.0], 0.1).scale_for(3)

    def test_raw_roundtrip_and_chain_rule(self):
        m = gp.KernelModel("matern32", 1.7, [0.3, 2.0, 0.9], 0.4, mean=-0.2, noise_floor=0.1)
        raw = gp.model_to_raw(m)
        m2 = gp.raw_to_model(m, raw)
        np.testing.assert_allclose(m2.lengthscales, m.lengthscales, rtol=1e-12)
        assert m2.noise == pytest.approx(m.noise, rel=1e-12)
        grads = {p: 1.0 for p in kernels.param_ids(m)}
        g = kernels.raw_gradient(m, raw, grads)
        h = 1e-6
        for i in range(raw.size - 1):
            e = np.zeros_like(raw)
            e[i] = h
            fd = (kernels.param_value(gp.raw_to_model(m, raw + e), kernels.param_ids(m)[i])
                  - kernels.param_value(gp.raw_to_model(m, raw - e), kernels.param_ids(m)[i])) / (2 * h)
            assert g[i] == pytest.approx(fd, rel=1e-6)
        assert g[-1] == 1.0

    def test_text_roundtrip(self, tmp_path):
        m = gp.KernelModel("rbf", 1.25, [0.5, 0.75], 0.3, mean=0.1, noise_floor=0.05)
        gp.save_model(m, tmp_path / "m.txt")
        m2 = gp.load_model(tmp_path / "m.txt")
        assert m2.family == m.family and m2.noise == m.noise
        np.testing.assert_array_equal(m2.lengthscales, m.lengthscales)
        with pytest.raises(ValueError):
            gp.model_from_text("family = rbf\n")


def test_cache_file_format_matches_reference_layout(tmp_path):
    """Byte layout of predictor.py:220-279: <BBQQQddddd + f64 arrays."""
    import struct
    rng = np.random.default_rng(0)
    m = gp.KernelModel("matern32", 1.5, [0.7, 1.1], 0.2, mean=0.3, noise_floor=0.1)
    X, w = rng.standard_normal((7, 2)), rng.standard_normal(7)
    c = predictor.PredictionCache(model=m, X_train=X, weights=w, cache_tolerance=1e-3)
    p = tmp_path / "c.bin"
    gp.save_cache(c, p)
    blob = p.read_bytes()
    head = struct.unpack_from("<BBQQQddddd", blob)
    assert head == (1, 1, 7, 2, 2, 1.5, 0.2, 0.1, 0.3, 1e-3)
    assert len(blob) == struct.calcsize("<BBQQQddddd") + 8 * (2 + 14 + 7)
    c2 = gp.load_cache(p)
    np.testing.assert_array_equal(c2.X_train, X)
    np.testing.assert_array_equal(c2.weights, w)
    with pytest.raises(ValueError):
        p.write_bytes(blob[:-8])
        gp.load_cache(p)


def test_cache_file_interoperates_with_reference(tmp_path):
    """A cache written here loads in the reference and vice versa (only in the
    build container, where /root/reference exists)."""
    if not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not present on this machine")
    import importlib
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        ref_pred = importlib.import_module("blockgp.predictor")
        ref_k = importlib.import_module("blockgp.kernels")
    finally:
        sys.path.remove("/root/reference/pkg/src")
    rng = np.random.default_rng(1)
    X, w = rng.standard_normal((5, 3)), rng.standard_normal(5)
    m = gp.KernelModel("rbf", 1.0, [0.5], 0.1)
    gp.save_cache(predictor.PredictionCache(m, X, w, 1e-3), tmp_path / "a.bin")
    rc = ref_pred.load_cache(tmp_path / "a.bin")
    np.testing.assert_array_equal(rc.weights, w)
    rm = ref_k.KernelModel("matern32", 2.0, np.array([0.4, 0.5, 0.6]), 0.3)
    ref_pred.save_cache(ref_pred.PredictionCache(rm, X, w, 1e-4), tmp_path / "b.bin")
    c = gp.load_cache(tmp_path / "b.bin")
    assert c.model.family == "matern32" and c.cache_tolerance == 1e-4
    np.testing.assert_array_equal(c.model.lengthscales, [0.4, 0.5, 0.6])


def test_solve_request_validation():
    with pytest.raises(ValueError):
        gp.SolveRequest(rhs=np.zeros((3, 2)), tolerance=1.0)
    with pytest.raises(ValueError):
        gp.SolveRequest(rhs=np.ones(3), tolerance=0.0)
    with pytest.raises(ValueError):
        gp.SolveRequest(rhs=np.ones(3), tolerance=1.0, max_iters=0)
    r = gp.SolveRequest(rhs=np.ones(3), tolerance=1.0)
    assert r.rhs.shape == (3, 1)


def test_tridiagonal_dense():
    T = gp.Tridiagonal(np.array([1.0, 2.0, 3.0]), np.array([0.5, 0.25]))
    np.testing.assert_array_equal(T.dense(), [[1, .5, 0], [.5, 2, .25], [0, .25, 3]])
    assert T.order == 3
