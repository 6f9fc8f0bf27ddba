"""Device residency helpers: host<->HBM transfers, the uploaded-input cache,
and prescaled point sets (X / lengthscale) in the layouts the kernels read."""

from __future__ import annotations

import weakref
import zlib
from collections import OrderedDict

import numpy as np

from . import _lib


def torch():
    import torch as _t
    return _t


_devices = {}


def device():
    """The current CUDA device (raises if the CUDA library or a device is
    missing)."""
    T = torch()
    idx = T._C._cuda_getDevice() if _devices else None
    dev = _devices.get(idx)
    if dev is None:
        _lib.lib()
        idx = T.cuda.current_device()
        dev = _devices[idx] = T.device("cuda", idx)
    return dev


def is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (float64 by default)."""
    T = torch()
    dtype = dtype or T.float64
    if is_tensor(x):
        t = x
        if t.device.type != "cuda":
            t = t.pin_memory().to(device(), non_blocking=True) if t.numel() > 4096 else t.to(device())
        return t.to(dtype).contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64 if dtype == T.float64 else None))
    t = T.from_numpy(a)
    if t.numel() > (1 << 16):
        t = t.pin_memory()
    return t.to(device(), non_blocking=True).to(dtype)


def to_host(t) -> np.ndarray:
    return t.detach().to("cpu").numpy()


class _UploadCache:
    """Keeps recently uploaded read-only host arrays (training inputs) in HBM
    so repeated MLL evaluations over the same X do not re-copy it. Keyed by
    the array object (weakref), its data pointer, shape and a CRC-32 of its
    full contents, so an in-place edit anywhere in the array invalidates the
    cached copy (≈4 GB/s on the host: 23 ms for a 10^6 x 11 array, less than
    the pinned staging copy of the upload it avoids)."""

    def __init__(self, capacity=4):
        self.capacity = capacity
        self.entries = OrderedDict()

    @staticmethod
    def _probe(a: np.ndarray):
        c = np.ascontiguousarray(a)
        return (c.shape, zlib.crc32(memoryview(c.reshape(-1)).cast("B")))

    def get(self, a, probe=None):
        if is_tensor(a):
            return to_device(a)
        a = np.asarray(a, dtype=np.float64)
        key = (id(a), a.__array_interface__["data"][0], a.shape, a.strides)
        if probe is None:
            probe = self._probe(a) if a.size else 0
        hit = self.entries.get(key)
        if hit is not None:
            ref, pr, t = hit
            if ref() is a and pr == probe:
                self.entries.move_to_end(key)
                return t
        t = to_device(a)
        try:
            ref = weakref.ref(a)
        except TypeError:  # pragma: no cover
            return t
        self.entries[key] = (ref, probe, t)
        while len(self.entries) > self.capacity:
            self.entries.popitem(last=False)
        return t


upload_cache = _UploadCache()


def ld32_for(d: int) -> int:
    return (d + 3) // 4 * 4


class PointSet:
    """Training/test inputs resident in HBM plus prescaled copies:
    Xs32 (n x ld32, fp32, zero padded) for the fused kernels and
    Xs64 (n x d, fp64) for the fp64 paths (pivoted Cholesky, dense blocks)."""

    def __init__(self, X, probe=None):
        X = upload_cache.get(X, probe)
        if X.dim() != 2:
            X = X.reshape(X.shape[0], -1)
        self.X = X
        self.n, self.d = X.shape
        self._scaled = {}

    def scaled(self, lengthscales):
        ls = np.atleast_1d(np.asarray(lengthscales, dtype=np.float64))
        key = ls.tobytes()
        hit = self._scaled.get(key)
        if hit is not None:
            return hit
        T = torch()
        if ls.size not in (1, self.d):
            raise ValueError(f"model has {ls.size} lengthscales but inputs have dimension {self.d}")
        ls_dev = T.from_numpy(ls.copy()).to(device())
        ld32 = ld32_for(self.d)
        Xs32 = T.empty((self.n, ld32), dtype=T.float32, device=device())
        Xs64 = T.empty((self.n, self.d), dtype=T.float64, device=device())
        L = _lib.lib()
        _lib.check(L.gp_prescale(_lib.ptr(self.X), self.n, self.d, self.d, _lib.ptr(ls_dev), ls.size,
                                 _lib.ptr(Xs32), ld32, _lib.ptr(Xs64), self.d, None,
                                 _lib.stream_handle()), "gp_prescale")
        if len(self._scaled) > 4:
            self._scaled.clear()
        self._scaled[key] = (Xs32, Xs64)
        return Xs32, Xs64


_points: "OrderedDict[int, PointSet]" = OrderedDict()


def points(X) -> PointSet:
    """PointSet for X, reusing the HBM copy (and its prescaled variants)
    across calls on the same, unmodified array."""
    if isinstance(X, PointSet):
        return X
    if is_tensor(X):
        return PointSet(X)
    a = np.asarray(X, dtype=np.float64)
    key = id(X)
    probe = _UploadCache._probe(a) if a.size else 0
    ps = _points.get(key)
    if ps is not None and ps._src() is X and ps._probe == probe:
        _points.move_to_end(key)
        return ps
    ps = PointSet(X, probe if a is X else None)
    try:
        ps._src = weakref.ref(X)
    except TypeError:
        return ps
    ps._probe = probe
    _points[key] = ps
    while len(_points) > 4:
        _points.popitem(last=False)
    return ps
