"""ctypes binding of libvqb200.so (the C ABI declared in include/vqb200.h).

Loading fails loudly: there is no CPU fallback for the hot path.  Status codes
map onto the reference's exception hierarchy (errors.py:8-29).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ConfigError, DomainError, FormatError, InternalError, UsageError

_HERE = os.path.dirname(os.path.abspath(__file__))
# VQB200_LIB: another build of the same ABI (A/B timing, profiling builds)
LIB_PATH = os.environ.get("VQB200_LIB") or os.path.join(_HERE, "libvqb200.so")

VQB_OK, VQB_USAGE, VQB_CONFIG, VQB_DOMAIN, VQB_INTERNAL, VQB_FORMAT = 0, 1, 2, 3, 4, 5

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_D = ctypes.c_double


class TrainConfig(ctypes.Structure):
    _fields_ = [
        ("target_size", ctypes.c_int64),
        ("epsilon", ctypes.c_double),
        ("delta", ctypes.c_double),
        ("max_iterations_per_level", ctypes.c_int64),
        ("metric", ctypes.c_int32),
        ("ordered", ctypes.c_int32),
        ("global_colmax", ctypes.c_void_p),   # const double[dim] or NULL
        ("global_collow", ctypes.c_void_p),   # const int32[dim] or NULL
    ]


class LevelIterationC(ctypes.Structure):
    _fields_ = [
        ("codebook_size", ctypes.c_int64),
        ("iteration", ctypes.c_int64),
        ("td", ctypes.c_double),
        ("empty_cells", ctypes.c_int64),
        ("seconds", ctypes.c_double),
    ]


class TrainSummary(ctypes.Structure):
    _fields_ = [
        ("total", ctypes.c_double),
        ("n_hist", ctypes.c_int64),
        ("n_warn", ctypes.c_int64),
        ("passes", ctypes.c_int64),
        ("flagged_rows", ctypes.c_int64),
        ("evals", ctypes.c_int64),
        ("final_size", ctypes.c_int64),
        ("fast_path", ctypes.c_int32),
        ("ordered", ctypes.c_int32),
        ("flagged_full", ctypes.c_int64),
        ("sums_exact", ctypes.c_int32),
        ("ref_exact", ctypes.c_int32),
    ]


_lib = None


def lib():
    """The loaded library (raises ImportError if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(make -C paper_0910_4711_b200/csrc); the B200 path has no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "vqb_last_error": ([], ctypes.c_char_p),
            "vqb_version": ([], _I32),
            "vqb_device_count": ([_P], _I32),
            "vqb_assign_range": ([_P, _I64, _I64, _P, _I64, _I64, _I64, _I32, _P, _P], _I32),
            "vqb_update_rows": ([_P, _I64, _I64, _P, _P, _I64, _I64, _I64, _P, _P], _I32),
            "vqb_column_sums": ([_P, _I64, _I64, _P], _I32),
            "vqb_sum_inorder": ([_P, _I64, _P], _I32),
            "vqb_pair_distance": ([_P, _P, _I64, _I32, _P], _I32),
            "vqb_split_codebook": ([_P, _I64, _I64, _D, _I32, _P], _I32),
            "vqb_open": ([_P, _P, _I64, _I64, _I64, _I64, _I32, _P], _I32),
            "vqb_close": ([_P], _I32),
            "vqb_set_stream": ([_P, _P], _I32),
            "vqb_local_maxabs": ([_P, _P], _I32),
            "vqb_local_colstats": ([_P, _P, _P], _I32),
            "vqb_session_info": ([_P, _P], _I32),
            "vqb_step_history": ([_P, _P, _I64, _P], _I32),
            "vqb_train": ([_P, _P, _P, _P, _I64, _P, _I64, _P, _P], _I32),
            "vqb_assign": ([_P, _P, _I64, _I32, _P, _P, _P, _P], _I32),
            "vqb_update": ([_P, _P, _P, _I64, _P, _P, _P], _I32),
            "vqb_step_begin": ([_P, _P], _I32),
            "vqb_step_local": ([_P], _I32),
            "vqb_step_finalize": ([_P], _I32),
            "vqb_step_exchange": ([_P, _P, _P], _I32),
            "vqb_step_poll": ([_P, _P], _I32),
            "vqb_step_result": ([_P, _P, _P, _I64, _P, _I64, _P, _P], _I32),
            "vqb_encode_f32": ([_P, _I64, _I64, _P, _I64, _I32, _P, _P], _I32),
            "vqb_lloyd_step_f32": ([_P, _I64, _I64, _P, _I64, _I32, _P, _P, _P, _P], _I32),
            "vqb_pipe_microbench": ([_I32, _I32, _I32, _P, _P], _I32),
            "vqb_bench_iteration": ([_P, _P, _I64, _I32, _P, _P], _I32),
            "vqb_bench_assign": ([_P, _P, _I64, _I32, _P, _P, _P], _I32),
            "vqb_bench_upload": ([_P, _I64, _I32, _P], _I32),
            "vqb_debug_tc_tile": ([_P, _P, _I64, _P, _P], _I32),
            "vqb_pixels_to_blocks": ([_P, _I64, _I64, _I64, _I64, _I32, _P, _P], _I32),
            "vqb_blocks_to_pixels": ([_P, _I64, _I64, _I64, _I64, _I32, _P], _I32),
            "vqb_decode": ([_P, _I64, _P, _I64, _I64, _I32, _P], _I32),
            "vqb_decode_pixels": ([_P, _I64, _I64, _I64, _I64, _P, _I64, _I32, _P], _I32),
            "vqb_reconstruction_distortion": ([_P, _P, _I64, _I64, _I32, _I32, _P], _I32),
            "vqb_open_pixels": ([_P, _I64, _I64, _I64, _I64, _I32, _P], _I32),
            "vqb_open_gmm": ([_P, _P, _P, _I64, _I64, _I64, _I64, _I64, ctypes.c_uint64, _I32, _P], _I32),
            "vqb_rows_f32": ([_P, _P], _I32),
            "vqb_host_copy": ([_P, _P, _I64], _I32),
            "vqb_lloyd_begin": ([_P, _P, _I64, _P, _P], _I32),
            "vqb_lloyd_local": ([_P], _I32),
            "vqb_first_nonfinite_f32": ([_P, _I64, _P], _I32),
            "vqb_first_nonfinite_f64": ([_P, _I64, _P], _I32),
            "vqb_bench_formats": ([_I32, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _P, _P], _I32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Raise the reference's exception class for a non-zero status."""
    if rc == VQB_OK:
        return
    msg = lib().vqb_last_error().decode(errors="replace")
    if rc == VQB_CONFIG:
        raise ConfigError(msg)
    if rc == VQB_USAGE:
        raise UsageError(msg)
    if rc == VQB_DOMAIN:
        raise DomainError(msg)
    if rc == VQB_FORMAT:
        raise FormatError(msg)
    raise InternalError(msg)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = lib().vqb_device_count(ctypes.byref(c))
    return int(c.value) if rc == VQB_OK else 0


def require_device() -> None:
    if device_count() < 1:
        raise InternalError("no CUDA device: the B200 hot path has no CPU fallback")
