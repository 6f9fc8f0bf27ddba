"""Device-side splitting / whitening / subset gathers (csrc/data.cu) against
the reference's split_and_whiten output (tests/golden/whiten.npz) and the
oracle (data.py:163-196, trainer.py:323-330)."""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_split_and_whiten_matches_reference():
    from paper_1903_08114_b200 import data
    g = load_golden("whiten")
    ds = data.split_and_whiten(data.RawTable(g["X_raw"], g["y_raw"]), int(g["seed"]), name="w")
    for a, b in ((ds.train_idx, g["train_idx"]), (ds.val_idx, g["val_idx"]), (ds.test_idx, g["test_idx"])):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_allclose(ds.feature_mean, g["feature_mean"], rtol=1e-14, atol=1e-12)
    np.testing.assert_allclose(ds.feature_std, g["feature_std"], rtol=1e-13)
    assert ds.feature_std[3] == 1.0
    assert ds.target_mean == pytest.approx(float(g["target_mean"]), rel=1e-14)
    assert ds.target_std == pytest.approx(float(g["target_std"]), rel=1e-13)
    # column 4 sits at 1e4 with spread 5: x - mean cancels ~11 bits, so the
    # last-bit difference of the two means shows up at ~2e-12 absolute
    np.testing.assert_allclose(ds.X, g["X"], rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(ds.y, g["y"], rtol=1e-12, atol=1e-12)
    # the standardized copies stay resident; the train split gathers on the device
    Xt, yt = ds.train_device()
    np.testing.assert_array_equal(Xt.cpu().numpy(), ds.X_train)
    np.testing.assert_array_equal(yt.cpu().numpy(), ds.y_train)
    sub = ds.subsample_train(0.25, 3)
    order = np.random.default_rng(3).permutation(ds.train_idx.shape[0])
    keep = max(1, int(round(0.25 * ds.train_idx.shape[0])))
    np.testing.assert_array_equal(sub.train_idx, np.sort(ds.train_idx[order[:keep]]))


def test_column_moments_and_gather_edges():
    from paper_1903_08114_b200 import data
    rng = np.random.default_rng(4)
    for n, d in ((1, 1), (7, 3), (70_000, 11), (513, 300)):
        A = rng.standard_normal((n, d)) * 10.0 ** rng.uniform(-3, 3, size=d) + rng.uniform(-5, 5, size=d)
        A[:, 0] = 2.0   # constant column
        rows = np.sort(rng.choice(n, size=max(1, n // 3), replace=False))
        mean, std = data.column_moments(A, rows)
        np.testing.assert_allclose(mean.cpu().numpy(), A[rows].mean(axis=0), rtol=1e-13, atol=1e-13)
        ref_std = A[rows].std(axis=0)
        ref_std[ref_std == 0.0] = 1.0
        np.testing.assert_allclose(std.cpu().numpy(), ref_std, rtol=1e-12, atol=1e-15)
        np.testing.assert_array_equal(data.gather_rows(A, rows).cpu().numpy(), A[rows])
    with pytest.raises(IndexError):
        data.gather_rows(np.zeros((4, 2)), [0, 4])
    with pytest.raises(ValueError):
        data.split_indices(8, 0)


def test_oracle_and_device_whitening_agree_at_scale():
    """n = 10^6 x 11 (the metric's shape): device statistics vs the oracle's."""
    from paper_1903_08114_b200 import data
    rng = np.random.default_rng(8)
    X = rng.uniform(-3, 7, size=(1_000_000, 11))
    y = rng.standard_normal(1_000_000)
    ds = data.split_and_whiten(data.RawTable(X, y), 9)
    Xs, ys, tr, va, te, fm, fs, tm, ts = O.split_and_whiten(X, y, 9)
    np.testing.assert_array_equal(ds.train_idx, tr)
    np.testing.assert_allclose(ds.feature_mean, fm, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(ds.feature_std, fs, rtol=1e-12)
    np.testing.assert_allclose(ds.X, Xs, rtol=1e-11, atol=1e-12)
