"""Splitting and whitening for the training protocol, statistics on the
device (data.py:17-196 of the reference).

The seeded shuffle and the split sizes are the reference's (host PCG64
permutation, 4/9 train, 2/9 validation, rest test); the training-split column
means and population standard deviations and the standardisation of every row
run as CUDA kernels (csrc/data.cu, gp_column_moments / gp_standardize), as does
the pretraining subset gather (gp_gather_rows, trainer.py:323-330). CSV
ingestion and the synthetic prior draw stay out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .kernels import KernelModel

SPLIT_NINTHS = (4, 2, 3)  # train, validation, test (data.py:20)


@dataclass
class RawTable:
    """Parsed table before splitting (data.py:25-33)."""

    features: np.ndarray
    target: np.ndarray
    feature_names: list = field(default_factory=list)
    target_name: str = "target"
    constant_columns: list = field(default_factory=list)


@dataclass
class Dataset:
    """A standardized dataset with its split and whitening record
    (data.py:36-100). X and y are host arrays (the reference's contract);
    `X_device` / `y_device` keep the standardized copies in HBM, where the
    likelihood and predictions consume them without another upload."""

    name: str
    X: np.ndarray
    y: np.ndarray
    train_idx: np.ndarray
    val_idx: np.ndarray
    test_idx: np.ndarray
    feature_mean: np.ndarray
    feature_std: np.ndarray
    target_mean: float
    target_std: float
    truth: KernelModel | None = None
    X_device: object = field(default=None, repr=False, compare=False)
    y_device: object = field(default=None, repr=False, compare=False)

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def d(self) -> int:
        return self.X.shape[1]

    @property
    def X_train(self):
        return self.X[self.train_idx]

    @property
    def y_train(self):
        return self.y[self.train_idx]

    @property
    def X_val(self):
        return self.X[self.val_idx]

    @property
    def y_val(self):
        return self.y[self.val_idx]

    @property
    def X_test(self):
        return self.X[self.test_idx]

    @property
    def y_test(self):
        return self.y[self.test_idx]

    def train_device(self):
        """(X_train, y_train) gathered on the device from the resident copies."""
        return gather_rows(self.X_device, self.train_idx), gather_rows(self.y_device[:, None], self.train_idx)[:, 0]

    def subsample_train(self, fraction: float, seed: int) -> "Dataset":
        """Nested seeded subset of the training split (data.py:84-100)."""
        if not 0 < fraction <= 1:
            raise ValueError("fraction must be in (0, 1]")
        rng = np.random.default_rng(seed)
        order = rng.permutation(self.train_idx.shape[0])
        keep = max(1, int(round(fraction * self.train_idx.shape[0])))
        sub = np.sort(self.train_idx[order[:keep]])
        return Dataset(name=f"{self.name}[{fraction:g}]", X=self.X, y=self.y, train_idx=sub,
                       val_idx=self.val_idx, test_idx=self.test_idx, feature_mean=self.feature_mean,
                       feature_std=self.feature_std, target_mean=self.target_mean,
                       target_std=self.target_std, truth=self.truth, X_device=self.X_device,
                       y_device=self.y_device)


def column_moments(A, rows=None, unit_if_zero: bool = True):
    """(mean, population std) per column of the device matrix A over `rows`
    (all rows when None), fp64 on the device; a zero std reads 1 when
    unit_if_zero (data.py:184-189)."""
    T = D.torch()
    A = D.to_device(A)
    if A.dim() == 1:
        A = A[:, None]
    n, d = A.shape
    if rows is not None:
        r = D.to_device(np.asarray(rows, dtype=np.int64), dtype=T.int64)
        m = int(r.shape[0])
    else:
        r, m = None, n
    if m < 1:
        raise ValueError("column moments of an empty row set")
    lib = _lib.lib()
    wl = int(lib.gp_column_moments_workspace_len(m, d))
    ws = T.empty(wl, dtype=T.float64, device=D.device())
    mean = T.empty(d, dtype=T.float64, device=D.device())
    std = T.empty(d, dtype=T.float64, device=D.device())
    _lib.check(lib.gp_column_moments(_lib.ptr(A), A.stride(0), m, d, _lib.ptr(r) if r is not None else 0,
                                     _lib.ptr(mean), _lib.ptr(std), int(unit_if_zero), _lib.ptr(ws), wl,
                                     _lib.stream_handle()), "gp_column_moments")
    return mean, std


def standardize(A, mean, std):
    """(A - mean) / std row-wise on the device (data.py:191-194)."""
    T = D.torch()
    A = D.to_device(A)
    vec = A.dim() == 1
    if vec:
        A = A[:, None]
    n, d = A.shape
    out = T.empty((n, d), dtype=T.float64, device=D.device())
    _lib.check(_lib.lib().gp_standardize(_lib.ptr(A), A.stride(0), n, d, _lib.ptr(mean), _lib.ptr(std),
                                         _lib.ptr(out), d, _lib.stream_handle()), "gp_standardize")
    return out[:, 0] if vec else out


def gather_rows(A, idx):
    """A[idx] for a device matrix A (or vector) and host/device indices."""
    T = D.torch()
    A = D.to_device(A)
    vec = A.dim() == 1
    if vec:
        A = A[:, None]
    n, d = A.shape
    ii = D.to_device(np.asarray(idx, dtype=np.int64) if not D.is_tensor(idx) else idx, dtype=T.int64)
    m = int(ii.shape[0])
    out = T.empty((m, d), dtype=T.float64, device=D.device())
    bad = T.zeros(1, dtype=T.int32, device=D.device())
    _lib.check(_lib.lib().gp_gather_rows(_lib.ptr(A), A.stride(0), n, _lib.ptr(ii), m, d, _lib.ptr(out), d,
                                         _lib.ptr(bad), _lib.stream_handle()), "gp_gather_rows")
    if m and int(bad.item()):
        raise IndexError("row index out of range")
    return out[:, 0] if vec else out


def split_indices(n: int, seed: int):
    """Seeded 4/9 : 2/9 : rest split of range(n), each part sorted
    (data.py:168-178)."""
    if n < 9:
        raise ValueError(f"need at least 9 rows to split, got {n}")
    order = np.random.default_rng(seed).permutation(n)
    n_train = (SPLIT_NINTHS[0] * n) // 9
    n_val = (SPLIT_NINTHS[1] * n) // 9
    return (np.sort(order[:n_train]), np.sort(order[n_train:n_train + n_val]),
            np.sort(order[n_train + n_val:]))


def split_and_whiten(raw: RawTable, seed: int, name: str = "dataset",
                     truth: KernelModel | None = None) -> Dataset:
    """Seeded split, then standardisation of every row by training-split
    statistics, computed on the device (data.py:163-196)."""
    X = np.atleast_2d(np.asarray(raw.features, dtype=np.float64))
    y = np.asarray(raw.target, dtype=np.float64)
    n = X.shape[0]
    train_idx, val_idx, test_idx = split_indices(n, seed)
    Xd, yd = D.to_device(X), D.to_device(y)
    f_mean, f_std = column_moments(Xd, train_idx, unit_if_zero=True)
    t_mean, t_std = column_moments(yd, train_idx, unit_if_zero=True)
    Xs = standardize(Xd, f_mean, f_std)
    ys = standardize(yd, t_mean, t_std)
    return Dataset(name=name, X=D.to_host(Xs), y=D.to_host(ys), train_idx=train_idx, val_idx=val_idx,
                   test_idx=test_idx, feature_mean=D.to_host(f_mean), feature_std=D.to_host(f_std),
                   target_mean=float(D.to_host(t_mean)[0]), target_std=float(D.to_host(t_std)[0]),
                   truth=truth, X_device=Xs, y_device=ys)
