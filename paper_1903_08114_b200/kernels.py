"""Kernel models and device-side kernel blocks (mirror of blockgp.kernels).

Host side keeps the reference's hyperparameter container and softplus
transforms (kernels.py:26-195; O(d) scalars). Everything that touches n
points runs on the GPU:
  * kernel_block / kernel_rows / kernel_eval -> gp_kernel_block (fp64)
  * training_mvm_oracle / cross_mvm_oracle return *descriptors*: called as
    row oracles they materialise blocks on the device, and
    partition.partitioned_mvm recognises them and runs the fused
    on-the-fly K·V kernel (gp_kv) instead, never forming the block.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _device as D
from . import _lib

FAMILIES = ("rbf", "matern32")
SQRT3 = float(np.sqrt(3.0))


@dataclass(frozen=True)
class KernelModel:
    """RBF or Matern-3/2 kernel with outputscale s2, shared (1,) or ARD (d,)
    lengthscales, Gaussian noise variance >= noise_floor, constant mean
    (same fields and validation as kernels.py:26-76)."""

    family: str
    outputscale: float
    lengthscales: np.ndarray
    noise: float
    mean: float = 0.0
    noise_floor: float = 0.0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown kernel family {self.family!r}")
        ls = np.array(np.atleast_1d(np.asarray(self.lengthscales, dtype=np.float64)))
        ls.setflags(write=False)
        object.__setattr__(self, "lengthscales", ls)
        checks = [(bool(np.all(ls > 0)), "lengthscales must be positive"),
                  (self.outputscale > 0, "outputscale must be positive"),
                  (self.noise_floor >= 0, "noise_floor must be non-negative"),
                  (self.noise >= self.noise_floor,
                   f"noise {self.noise} is below the floor {self.noise_floor}")]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def ard(self) -> bool:
        return self.lengthscales.size > 1

    def scale_for(self, d: int) -> np.ndarray:
        if self.ard and self.lengthscales.size != d:
            raise ValueError(f"model has {self.lengthscales.size} lengthscales "
                             f"but inputs have dimension {d}")
        return self.lengthscales

    @property
    def family_code(self) -> int:
        return _lib.FAMILY_CODE[self.family]


def default_model(family: str, d: int, *, ard: bool = False, noise_floor: float = 0.0,
                  target_mean: float = 0.0) -> KernelModel:
    """Pre-training initialisation (kernels.py:79-91): s2 = 1, l = 1,
    noise = max(1, floor + 0.5), mean = target mean."""
    return KernelModel(family, 1.0, np.ones(d if ard else 1), max(1.0, noise_floor + 0.5),
                       mean=float(target_mean), noise_floor=noise_floor)


# --- unconstrained parameterisation (kernels.py:97-195) --------------------
# raw vector layout: [s2, l..., noise - floor, mean], positives via softplus

def softplus(x):
    return np.logaddexp(0.0, x)


def inv_softplus(y):
    y = np.asarray(y, dtype=np.float64)
    if np.any(y <= 0):
        raise ValueError("inv_softplus requires positive input")
    return y + np.log(-np.expm1(-y))


def _dsoftplus(x):
    return 0.5 * (1.0 + np.tanh(0.5 * np.asarray(x, dtype=np.float64)))


def param_ids(model: KernelModel) -> list[str]:
    ls = ([f"lengthscale_{i}" for i in range(model.lengthscales.size)] if model.ard
          else ["lengthscale"])
    return ["outputscale", *ls, "noise", "mean"]


def _ls_index(pid: str) -> int | None:
    if pid == "lengthscale":
        return 0
    if pid.startswith("lengthscale_"):
        return int(pid.split("_", 1)[1])
    return None


def param_value(model: KernelModel, pid: str) -> float:
    if pid in ("outputscale", "noise", "mean"):
        return float(getattr(model, pid))
    i = _ls_index(pid)
    if i is None:
        raise ValueError(f"unknown hyperparameter {pid!r}")
    return float(model.lengthscales[i])


def with_param(model: KernelModel, pid: str, value: float) -> KernelModel:
    if pid in ("outputscale", "noise", "mean"):
        return replace(model, **{pid: value})
    i = _ls_index(pid)
    if i is None:
        raise ValueError(f"unknown hyperparameter {pid!r}")
    ls = model.lengthscales.copy()
    if pid == "lengthscale":
        ls = np.array([value])
    else:
        ls[i] = value
    return replace(model, lengthscales=ls)


def model_to_raw(model: KernelModel) -> np.ndarray:
    return np.concatenate([[inv_softplus(model.outputscale)], inv_softplus(model.lengthscales),
                           [inv_softplus(model.noise - model.noise_floor)], [model.mean]]).astype(np.float64)


def raw_to_model(template: KernelModel, raw) -> KernelModel:
    raw = np.asarray(raw, dtype=np.float64)
    m = template.lengthscales.size
    if raw.shape != (m + 3,):
        raise ValueError(f"raw vector has shape {raw.shape}, expected ({m + 3},)")
    return replace(template, outputscale=float(softplus(raw[0])),
                   lengthscales=softplus(raw[1:1 + m]),
                   noise=template.noise_floor + float(softplus(raw[1 + m])),
                   mean=float(raw[2 + m]))


def raw_gradient(model: KernelModel, raw, grads: dict) -> np.ndarray:
    """Chain rule through the softplus transforms (kernels.py:182-195)."""
    raw = np.asarray(raw, dtype=np.float64)
    ids = param_ids(model)
    out = np.array([grads[p] for p in ids], dtype=np.float64)
    out[:-1] *= _dsoftplus(raw[:-1])
    return out


# --- device kernel blocks ----------------------------------------------------

def _dense_block(model: KernelModel, Xr_ps: D.PointSet, Xc_ps: D.PointSet, diag_offset: int,
                 row_slice=None):
    """fp64 kernel block on the device (optionally a row slice of Xr)."""
    T = D.torch()
    ls = model.scale_for(Xr_ps.d)
    _, Xr64 = Xr_ps.scaled(ls)
    _, Xc64 = Xc_ps.scaled(ls) if Xc_ps is not Xr_ps else (None, Xr64)
    if row_slice is not None:
        Xr64 = Xr64[row_slice[0]:row_slice[1]]
    nr, nc = Xr64.shape[0], Xc64.shape[0]
    out = T.empty((nr, nc), dtype=T.float64, device=D.device())
    _lib.check(_lib.lib().gp_kernel_block(model.family_code, Xr_ps.d, _lib.ptr(Xr64), Xr_ps.d, nr,
                                          _lib.ptr(Xc64), Xc_ps.d, nc, float(model.outputscale),
                                          float(model.noise), int(diag_offset), _lib.ptr(out), nc,
                                          _lib.stream_handle()), "gp_kernel_block")
    return out


def _as_points(X):
    if isinstance(X, D.PointSet) or D.is_tensor(X):
        return D.points(X)
    return D.points(np.atleast_2d(np.asarray(X, dtype=np.float64)))


def _pointsets(X_rows, X_cols):
    Xr, Xc = _as_points(X_rows), _as_points(X_cols)
    if Xr.d != Xc.d:
        raise ValueError(f"dimension mismatch: rows have d={Xr.d}, cols have d={Xc.d}")
    return Xr, Xc


def kernel_eval(model: KernelModel, x, xp) -> float:
    """k(x, x') (kernels.py:202-213)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    xp = np.atleast_1d(np.asarray(xp, dtype=np.float64))
    if x.shape != xp.shape:
        raise ValueError(f"point dimensions differ: {x.shape} vs {xp.shape}")
    return float(kernel_block(model, x[None, :], xp[None, :])[0, 0])


def kernel_block_device(model: KernelModel, X_rows, X_cols, add_noise: bool = False):
    Xr, Xc = _pointsets(X_rows, X_cols)
    if add_noise and Xr.n != Xc.n:
        raise ValueError("noise can only be added to the square training block")
    return _dense_block(model, Xr, Xc, 0 if add_noise else -1)


def kernel_block(model: KernelModel, X_rows, X_cols, add_noise: bool = False) -> np.ndarray:
    """Dense fp64 kernel block (kernels.py:247-270), computed on the GPU."""
    return D.to_host(kernel_block_device(model, X_rows, X_cols, add_noise))


def kernel_rows(model: KernelModel, X, start: int, stop: int, *, noise: bool = True) -> np.ndarray:
    """Rows [start, stop) of the (noise-augmented) training matrix
    (kernels.py:293-308), computed on the GPU."""
    ps = D.points(X)
    model.scale_for(ps.d)
    return D.to_host(_dense_block(model, ps, ps, start if noise else -1, (start, stop)))


class TrainingOperator:
    """Descriptor of K̂ = K(X,X) + noise I for the partitioned executor
    (kernels.py:311-316). As a callable it returns materialised rows like the
    reference row oracle; partitioned_mvm runs gp_kv on it instead."""

    def __init__(self, model: KernelModel):
        self.model = model

    def __call__(self, X, start, stop):
        return kernel_rows(self.model, X, start, stop, noise=True)


class CrossOperator:
    """Descriptor of K(X_rows, X_cols) without noise (kernels.py:319-325)."""

    def __init__(self, model: KernelModel, X_cols):
        self.model = model
        self.X_cols = X_cols

    def __call__(self, X, start, stop):
        Xr = np.asarray(X)[start:stop] if not D.is_tensor(X) else X[start:stop]
        return kernel_block(self.model, Xr, self.X_cols)


def training_mvm_oracle(model: KernelModel) -> TrainingOperator:
    return TrainingOperator(model)


def cross_mvm_oracle(model: KernelModel, X_cols) -> CrossOperator:
    return CrossOperator(model, X_cols)


def kernel_block_grad(model: KernelModel, X_rows, X_cols, param: str) -> np.ndarray:
    """dK/dtheta block for one constrained hyperparameter (kernels.py:374-393).
    Off the hot path (the MLL uses gp_grad_forms); computed on the device
    from the fp64 kernel block."""
    Xr, Xc = _pointsets(X_rows, X_cols)
    T = D.torch()
    if param == "noise":
        out = T.zeros((Xr.n, Xc.n), dtype=T.float64, device=D.device())
        if Xr.n == Xc.n:
            out.fill_diagonal_(1.0)
        return D.to_host(out)
    if param == "mean":
        raise ValueError("the mean has no kernel-block derivative")
    i = _ls_index(param)
    if param != "outputscale" and i is None:
        raise ValueError(f"unknown hyperparameter {param!r}")
    ls = model.scale_for(Xr.d)
    K = _dense_block(model, Xr, Xc, -1)
    if param == "outputscale":
        return D.to_host(K / model.outputscale)
    _, A = Xr.scaled(ls)
    _, B = Xc.scaled(ls)
    Dsq = T.cdist(A, B).square_()
    if model.family == "rbf":
        env = K
    else:
        env = 3.0 * model.outputscale * T.exp(-SQRT3 * Dsq.sqrt())
    if param == "lengthscale":
        return D.to_host(env * Dsq / float(ls[0]))
    if not model.ard:
        raise ValueError(f"unknown hyperparameter {param!r}")
    diff = (A[:, i, None] - B[None, :, i]) ** 2
    return D.to_host(env * diff / float(ls[i]))


def grad_row_products(model: KernelModel, X, start, stop, R, pids) -> dict:
    """(dK/dtheta)[start:stop, :] @ R per geometric parameter
    (kernels.py:396-410) — API compatibility only; the MLL uses the fused
    gp_grad_forms path."""
    X = np.asarray(X, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    return {p: kernel_block_grad(model, X[start:stop], X, p) @ R for p in pids}


# --- text persistence (kernels.py:417-464) -----------------------------------

def model_to_text(model: KernelModel) -> str:
    rows = [("family", model.family), ("num_lengthscales", str(model.lengthscales.size)),
            ("outputscale", repr(model.outputscale)),
            ("lengthscales", " ".join(repr(float(v)) for v in model.lengthscales)),
            ("noise", repr(model.noise)), ("noise_floor", repr(model.noise_floor)),
            ("mean", repr(model.mean))]
    return "".join(f"{k} = {v}\n" for k, v in rows)


def model_from_text(text: str) -> KernelModel:
    fields = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        key, sep, value = line.partition("=")
        if not sep:
            raise ValueError(f"line {lineno}: expected 'key = value'")
        fields[key.strip()] = value.strip()
    try:
        ls = np.array([float(v) for v in fields["lengthscales"].split()])
        model = KernelModel(fields["family"], float(fields["outputscale"]), ls,
                            float(fields["noise"]), mean=float(fields["mean"]),
                            noise_floor=float(fields["noise_floor"]))
    except KeyError as exc:
        raise ValueError(f"missing model field {exc.args[0]!r}") from exc
    if int(fields["num_lengthscales"]) != ls.size:
        raise ValueError("lengthscale count disagrees with num_lengthscales")
    return model


def save_model(model: KernelModel, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(model_to_text(model))


def load_model(path) -> KernelModel:
    with open(path, "r", encoding="ascii") as fh:
        return model_from_text(fh.read())
