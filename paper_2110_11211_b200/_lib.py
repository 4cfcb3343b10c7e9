"""ctypes binding of libsfcdd_b200.so (the C ABI in include/sfcdd_b200.h).

This is exactly the binding a maintainer of the reference would add on the
reference side: plain pointers, sizes and int status codes.
The library is built in-tree by ``paper_2110_11211_b200.build``; if it is
missing, importing any compute module fails loudly -- there is no CPU
fallback for the hot path.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

# SFCDD_LIB: alternative build of the same library (A/B timing of kernel variants)
_LIB_PATH = Path(os.environ.get("SFCDD_LIB") or Path(__file__).resolve().parent / "libsfcdd_b200.so")

SFCDD_OK = 0
SFCDD_EVALUE = -1
SFCDD_EFACTOR = -2
SFCDD_EBREAKDOWN = -3
SFCDD_EOVERFLOW = -4
SFCDD_ECUDA = -5
SFCDD_EINTERNAL = -6

VARIANT_CODES = {"one_level": 0, "additive_two_level": 1, "deflated": 2, "balanced": 3}
WEIGHTING_CODES = {"none": 0, "omega": 1, "d_matrix": 2}


class FactorizationError(RuntimeError):
    """Raised when a matrix expected to be SPD cannot be factorized (linalg.py:21)."""


class BreakdownError(RuntimeError):
    """Nonpositive curvature encountered in a CG recurrence (krylov.py:21)."""


class DivergenceError(RuntimeError):
    """Richardson error grew by 10x over its initial value (krylov.py:25)."""


class DeviceError(RuntimeError):
    """CUDA runtime failure (no device, launch failure, out of memory)."""


CURVES = {"hilbert": 0, "lebesgue": 1}


class OpDesc(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("levels", ctypes.c_int32 * 8),
        ("p", ctypes.c_int32),
        ("q", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("weighting", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("ov_start", ctypes.c_void_p),
        ("ov_len", ctypes.c_void_p),
        ("dj_start", ctypes.c_void_p),
        ("dj_len", ctypes.c_void_p),
        ("omega", ctypes.c_void_p),
        ("host_threads", ctypes.c_int32),
        ("shard_first", ctypes.c_int32),
        ("shard_count", ctypes.c_int32),
        ("curve", ctypes.c_int32),
        ("raw_laplacian", ctypes.c_int32),
        ("gamma_num", ctypes.c_int64),
        ("gamma_den", ctypes.c_int64),
        ("reserved", ctypes.c_int32 * 4),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("n0", ctypes.c_int64),
        ("factor_nnz", ctypes.c_int64),
        ("factor_nnz_l", ctypes.c_int64),
        ("coarse_nnz", ctypes.c_int64),
        ("num_tasks", ctypes.c_int64),
        ("num_supernodes", ctypes.c_int64),
        ("setup_seconds", ctypes.c_double),
        ("order_seconds", ctypes.c_double),
        ("factor_seconds", ctypes.c_double),
        ("apply_calls", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
        ("last_solve_ms", ctypes.c_double),
        ("reserved", ctypes.c_int64 * 8),
    ]


EXPORTS = [
    "sfcdd_last_error", "sfcdd_version", "sfcdd_sfc_encode", "sfcdd_sfc_decode",
    "sfcdd_sfc_perm", "sfcdd_sfc_encode_curve", "sfcdd_sfc_decode_curve", "sfcdd_sfc_perm_curve", "sfcdd_op_create", "sfcdd_op_setup", "sfcdd_op_apply",
    "sfcdd_op_matvec", "sfcdd_op_pcg", "sfcdd_op_pcg_ex", "sfcdd_vec_dot", "sfcdd_vec_axpby",
    "sfcdd_op_set_fault", "sfcdd_op_reset_calls",
    "sfcdd_op_stats", "sfcdd_op_stencil", "sfcdd_op_coarse_dense", "sfcdd_op_destroy",
    "sfcdd_op_profile", "sfcdd_op_trace",
    "sfcdd_shard_info", "sfcdd_op_neighbors", "sfcdd_shard_xy", "sfcdd_shard_residual", "sfcdd_shard_pm", "sfcdd_shard_update",
    "sfcdd_shard_coarse", "sfcdd_shard_tvec", "sfcdd_shard_local_solve", "sfcdd_shard_combine",
    "sfcdd_shard_stencil_restrict", "sfcdd_shard_finalize", "sfcdd_pack", "sfcdd_unpack",
    "sfcdd_factor_create", "sfcdd_factor_solve", "sfcdd_factor_info", "sfcdd_factor_destroy",
    "sfcdd_host_amd", "sfcdd_host_factor_solve", "sfcdd_host_plan_solve",
    "sfcdd_partition", "sfcdd_partition_weights", "sfcdd_csr_create", "sfcdd_csr_matvec", "sfcdd_csr_destroy",
    "sfcdd_host_setup_timing", "sfcdd_host_plan_deferred_check",
    "sfcdd_nccl_unique_id", "sfcdd_shard_attach", "sfcdd_shard_set_exchange", "sfcdd_shard_pcg",
]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing; build it with `python -m paper_2110_11211_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(str(_LIB_PATH))
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.sfcdd_last_error.restype = ctypes.c_char_p
    L.sfcdd_version.restype = ctypes.c_int
    sigs = {
        "sfcdd_sfc_encode": [ctypes.c_int, ctypes.c_int, vp, i64, vp, vp, vp],
        "sfcdd_sfc_decode": [ctypes.c_int, ctypes.c_int, vp, vp, i64, vp, vp],
        "sfcdd_sfc_perm": [ctypes.c_int, vp, vp, vp, ctypes.c_int, vp],
        "sfcdd_sfc_encode_curve": [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, i64, vp, vp, vp],
        "sfcdd_sfc_decode_curve": [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, i64, vp, vp],
        "sfcdd_sfc_perm_curve": [ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int, vp],
        "sfcdd_op_create": [ctypes.POINTER(OpDesc), ctypes.POINTER(vp)],
        "sfcdd_op_setup": [vp, vp],
        "sfcdd_op_apply": [vp, vp, vp, vp],
        "sfcdd_op_matvec": [vp, vp, vp, vp],
        "sfcdd_op_pcg": [vp, vp, vp, dbl, i32, vp, ctypes.POINTER(i32), ctypes.POINTER(i32), vp],
        "sfcdd_op_pcg_ex": [vp, vp, vp, vp, i32, dbl, i32, vp, vp, ctypes.POINTER(i32), ctypes.POINTER(i32), vp],
        "sfcdd_vec_dot": [vp, vp, i64, ctypes.POINTER(dbl), vp],
        "sfcdd_vec_axpby": [dbl, vp, dbl, vp, i64, vp],
        "sfcdd_op_set_fault": [vp, i64, vp, i32],
        "sfcdd_op_reset_calls": [vp],
        "sfcdd_op_stats": [vp, ctypes.POINTER(Stats)],
        "sfcdd_op_stencil": [vp, vp, vp, vp],
        "sfcdd_op_coarse_dense": [vp, vp],
        "sfcdd_op_profile": [vp, vp, vp, i32, vp, vp, vp],
        "sfcdd_op_trace": [vp, vp, vp, ctypes.POINTER(i64)],
        "sfcdd_shard_info": [vp, vp, vp],
        "sfcdd_op_neighbors": [vp, vp],
        "sfcdd_shard_xy": [vp, ctypes.POINTER(vp)],
        "sfcdd_shard_residual": [vp, vp, vp, vp, vp, vp, vp],
        "sfcdd_shard_pm": [vp, vp, vp, dbl, vp, vp, vp, vp],
        "sfcdd_shard_update": [vp, vp, vp, vp, vp, dbl, vp, vp, vp],
        "sfcdd_shard_coarse": [vp, vp, vp, vp],
        "sfcdd_shard_tvec": [vp, vp, vp, vp, vp],
        "sfcdd_shard_local_solve": [vp, vp, vp],
        "sfcdd_shard_combine": [vp, vp, vp],
        "sfcdd_shard_stencil_restrict": [vp, vp, vp, vp],
        "sfcdd_shard_finalize": [vp, vp, vp, vp, vp, vp, vp, vp],
        "sfcdd_pack": [vp, vp, i64, vp, vp],
        "sfcdd_unpack": [vp, vp, i64, vp, vp],
        "sfcdd_factor_create": [i64, vp, vp, vp, i32, ctypes.POINTER(vp)],
        "sfcdd_factor_solve": [vp, vp, vp, vp],
        "sfcdd_factor_info": [vp, vp, vp, vp],
        "sfcdd_host_amd": [i64, vp, vp, vp],
        "sfcdd_host_factor_solve": [i64, vp, vp, vp, vp, vp, vp, vp],
        "sfcdd_host_plan_solve": [i64, vp, vp, vp, i32, vp, vp, vp, vp, i32, i32, vp],
        "sfcdd_partition": [i64, i32, i64, i64, vp, vp, vp, vp],
        "sfcdd_partition_weights": [i64, i32, vp, vp, vp, vp],
        "sfcdd_csr_create": [i64, i64, vp, vp, vp, i32, ctypes.POINTER(vp)],
        "sfcdd_csr_matvec": [vp, vp, vp, vp],
        "sfcdd_host_setup_timing": [i64, vp, vp, vp, i32, vp, vp],
        "sfcdd_host_plan_deferred_check": [i64, vp, vp, vp, i32, vp, vp, vp, vp, vp],
        "sfcdd_nccl_unique_id": [vp],
        "sfcdd_shard_attach": [vp, vp, i32, i32, vp],
        "sfcdd_shard_set_exchange": [vp, i32, i32, vp, vp, vp, vp, vp],
        "sfcdd_shard_pcg": [vp, vp, vp, dbl, i32, vp, ctypes.POINTER(i32), ctypes.POINTER(i32), vp],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.sfcdd_op_destroy.argtypes = [vp]
    L.sfcdd_op_destroy.restype = None
    L.sfcdd_factor_destroy.argtypes = [vp]
    L.sfcdd_factor_destroy.restype = None
    L.sfcdd_csr_destroy.argtypes = [vp]
    L.sfcdd_csr_destroy.restype = None
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == SFCDD_OK:
        return
    msg = lib().sfcdd_last_error().decode(errors="replace")
    if rc == SFCDD_EVALUE:
        raise ValueError(msg)
    if rc == SFCDD_EFACTOR:
        raise FactorizationError(msg)
    if rc == SFCDD_EBREAKDOWN:
        raise BreakdownError(msg)
    if rc == SFCDD_EOVERFLOW:
        raise OverflowError(msg)
    if rc == SFCDD_ECUDA:
        raise DeviceError(msg)
    raise RuntimeError(f"sfcdd internal error ({rc}): {msg}")


def ptr(a) -> int:
    """Raw pointer of a numpy array or a torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def device():
    """The CUDA device used by the package (torch plumbing, fails loudly)."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the sfcdd B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def host_threads() -> int:
    return int(os.environ.get("SFCDD_HOST_THREADS", "0"))
