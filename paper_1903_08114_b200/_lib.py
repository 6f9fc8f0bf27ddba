"""ctypes binding of the C-ABI library (include/gpbbmm.h).

The product path has no CPU fallback: every entry point here runs a CUDA
kernel from the in-tree ``_lib/libgpbbmm.so``; if the library or a CUDA
device is missing, ``lib()`` raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NumericError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libgpbbmm.so")

GP_OK, GP_EINVAL, GP_ENONFINITE, GP_ENOTPD, GP_ECUDA, GP_EUNSUPPORTED = range(6)
FAMILY_CODE = {"rbf": 0, "matern32": 1}

c_i32, c_i64, c_f64, c_sz, c_p = C.c_int32, C.c_int64, C.c_double, C.c_size_t, C.c_void_p


class KvDesc(C.Structure):
    _fields_ = [("family", c_i32), ("d", c_i32),
                ("Xr", c_p), ("ldr", c_i64), ("n_rows", c_i64),
                ("Xc", c_p), ("ldc", c_i64), ("n_cols", c_i64),
                ("outputscale", c_f64), ("noise", c_f64), ("diag_offset", c_i64),
                ("algo", c_i32), ("reserved", c_i32), ("self_offset", c_i64)]


class MbcgState(C.Structure):
    _fields_ = [("n", c_i64), ("t", c_i32), ("k", c_i32), ("ld", c_i64), ("ld32", c_i64),
                ("U", c_p), ("R", c_p), ("P", c_p), ("Z", c_p), ("P32", c_p),
                ("noise", c_f64), ("L", c_p), ("ldl", c_i64), ("Binv", c_p), ("pc_noise", c_f64),
                ("bnorm", c_p), ("gamma", c_p), ("red", c_p), ("cbuf", c_p),
                ("alpha_hist", c_p), ("beta_hist", c_p), ("rel", c_p), ("rel_hist", c_p),
                ("active", c_p), ("converged", c_p), ("status", c_p),
                ("partials", c_p), ("partials_len", c_i64), ("max_iters", c_i32),
                ("nblocks", c_i32)]


_SIGS = {
    "gp_last_error": (C.c_char_p, []),
    "gp_version": (C.c_int, []),
    "gp_launch_count": (C.c_uint64, []),
    "gp_has_tcgen05": (C.c_int, []),
    "gp_prescale": (C.c_int, [c_p, c_i64, C.c_int, c_i64, c_p, C.c_int, c_p, c_i64, c_p, c_i64, c_p, c_p]),
    "gp_kv_workspace_bytes": (c_sz, [C.POINTER(KvDesc), C.c_int]),
    "gp_kv": (C.c_int, [C.POINTER(KvDesc), c_p, c_i64, C.c_int, c_p, c_i64, c_p, c_sz, c_p]),
    "gp_kv_sym_supported": (C.c_int, [C.POINTER(KvDesc), C.c_int]),
    "gp_kv_sym_auto": (C.c_int, [C.POINTER(KvDesc), C.c_int]),
    "gp_kv_sym_acc_ld": (c_i64, [C.POINTER(KvDesc)]),
    "gp_kv_sym_partial": (C.c_int, [C.POINTER(KvDesc), c_p, c_i64, C.c_int, C.c_int, C.c_int, c_p, c_p, c_p,
                                    c_sz, c_p]),
    "gp_kv_sym_finalize": (C.c_int, [C.POINTER(KvDesc), c_p, c_i64, C.c_int, c_p, c_p, c_i64, c_i64, c_i64,
                                     c_p, c_i64, c_p, c_sz, c_p]),
    "gp_kernel_block": (C.c_int, [C.c_int, C.c_int, c_p, c_i64, c_i64, c_p, c_i64, c_i64, c_f64,
                                  c_f64, c_i64, c_p, c_i64, c_p]),
    "gp_kv_f64_workspace_bytes": (c_sz, [c_i64, c_i64, C.c_int]),
    "gp_kv_f64": (C.c_int, [C.c_int, C.c_int, c_p, c_i64, c_i64, c_p, c_i64, c_i64, c_f64, c_f64, c_i64,
                            c_p, c_i64, C.c_int, c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "gp_block_mvm": (C.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_i64, C.c_int, c_p, c_i64, c_p, c_p]),
    "gp_mbcg_partials_len": (c_i64, [c_i64, C.c_int, C.c_int]),
    "gp_mbcg_init_a": (C.c_int, [C.POINTER(MbcgState), c_p, c_i64, c_p]),
    "gp_mbcg_init_b": (C.c_int, [C.POINTER(MbcgState), c_p]),
    "gp_mbcg_init_c": (C.c_int, [C.POINTER(MbcgState), c_p]),
    "gp_mbcg_pv": (C.c_int, [C.POINTER(MbcgState), c_p, c_i64, C.c_int, c_p]),
    "gp_mbcg_update": (C.c_int, [C.POINTER(MbcgState), c_p, c_i64, C.c_int, C.c_int, c_p]),
    "gp_mbcg_precond": (C.c_int, [C.POINTER(MbcgState), C.c_int, c_f64, c_p]),
    "gp_mbcg_direction": (C.c_int, [C.POINTER(MbcgState), C.c_int, c_p]),
    "gp_coldot": (C.c_int, [c_i64, C.c_int, c_p, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p]),
    "gp_lt_mul": (C.c_int, [c_i64, C.c_int, c_p, c_i64, c_p, c_i64, C.c_int, c_p, c_p, c_i64, c_p]),
    "gp_lowrank_mul": (C.c_int, [c_i64, C.c_int, c_p, c_i64, c_p, c_i64, C.c_int, c_f64, c_f64,
                                 c_p, c_i64, c_p]),
    "gp_pivchol_workspace_bytes": (c_sz, [c_i64, C.c_int]),
    "gp_pivchol": (C.c_int, [C.c_int, C.c_int, c_p, c_i64, c_i64, c_f64, C.c_int, c_p, c_i64, c_p,
                             c_p, c_p, c_p, c_sz, c_p]),
    "gp_precond_factor": (C.c_int, [c_i64, C.c_int, c_p, c_i64, c_f64, c_p, c_p, c_p, c_p, c_p,
                                    c_i64, c_p]),
    "gp_grad_forms_workspace_bytes": (c_sz, [c_i64, c_i64, C.c_int, C.c_int, C.c_int]),
    "gp_grad_forms": (C.c_int, [C.c_int, C.c_int, C.c_int, c_p, c_i64, c_i64, c_p, c_i64, c_i64,
                                c_f64, c_p, c_i64, c_p, c_i64, C.c_int, c_i64, C.c_int, c_p, c_p,
                                c_sz, c_p]),
    "gp_mbcg_solve_kv": (C.c_int, [C.POINTER(MbcgState), C.POINTER(KvDesc), c_p, c_i64, c_p, c_sz, c_f64,
                                   C.POINTER(c_i32), c_p]),
    "gp_column_moments_workspace_len": (c_i64, [c_i64, C.c_int]),
    "gp_column_moments": (C.c_int, [c_p, c_i64, c_i64, C.c_int, c_p, c_p, c_p, C.c_int, c_p, c_i64, c_p]),
    "gp_standardize": (C.c_int, [c_p, c_i64, c_i64, C.c_int, c_p, c_p, c_p, c_i64, c_p]),
    "gp_gather_rows": (C.c_int, [c_p, c_i64, c_i64, c_p, c_i64, C.c_int, c_p, c_i64, c_p, c_p]),
    "gp_comm_available": (C.c_int, []),
    "gp_comm_init": (C.c_int, [C.c_int, c_p, C.POINTER(c_p)]),
    "gp_comm_destroy": (C.c_int, [c_p]),
    "gp_comm_size": (C.c_int, [c_p]),
    "gp_comm_broadcast": (C.c_int, [c_p, c_p, c_i64, C.c_int, c_p]),
    "gp_comm_allgather": (C.c_int, [c_p, c_p, c_p, c_i64, c_p]),
    "gp_comm_reduce_scatter_i64": (C.c_int, [c_p, c_p, c_p, c_i64, c_p]),
    "gp_comm_reduce_scatter_i32": (C.c_int, [c_p, c_p, c_p, c_i64, c_p]),
    "gp_comm_allreduce_f64": (C.c_int, [c_p, c_p, c_i64, c_p]),
    "gp_grad_forms_sym_supported": (C.c_int, [c_i64, C.c_int, C.c_int, C.c_int]),
    "gp_grad_forms_sym_workspace_bytes": (c_sz, [c_i64, C.c_int, C.c_int, C.c_int]),
    "gp_grad_forms_sym": (C.c_int, [C.c_int, C.c_int, C.c_int, c_p, c_i64, c_i64, c_f64, c_p, c_i64, c_p,
                                    c_i64, C.c_int, c_p, c_p, c_sz, c_p]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare prototypes (no GPU needed)."""
    if not os.path.exists(path):
        raise RuntimeError(
            f"gpbbmm CUDA library not built at {path}; run `python -m "
            "paper_1903_08114_b200._build` (there is no CPU fallback)")
    so = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(so, name)
        fn.restype = res
        fn.argtypes = args
    return so


def lib():
    """The loaded library; raises loudly if it or a CUDA device is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch
                if not torch.cuda.is_available():
                    raise RuntimeError(
                        "paper_1903_08114_b200 needs a CUDA (sm_100a) device; "
                        "there is no CPU fallback")
                # GPBBMM_LIB: a variant build of the same library (A/B
                # diagnostics, scripts/build_variant.py); default in-tree
                _lib = load_library(os.environ.get("GPBBMM_LIB") or LIB_PATH)
    return _lib


def check(status: int, what: str = "") -> None:
    """Map a C status code to the reference's exception classes."""
    if status == GP_OK:
        return
    msg = (_lib.gp_last_error() or b"").decode(errors="replace") if _lib else ""
    if what:
        msg = f"{what}: {msg}"
    if status in (GP_EINVAL, GP_EUNSUPPORTED):
        raise ValueError(msg)
    if status in (GP_ENONFINITE, GP_ENOTPD):
        raise NumericError(msg)
    raise RuntimeError(msg)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    """The current CUDA stream of `device` (default: the current device) as
    a raw handle, without building a torch Stream object per call."""
    import torch
    if device is None:
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream(device).cuda_stream
