"""ctypes binding of libsinkattn.so (include/sinkattn.h).

The shared library is the product: every compute call goes through it.  If it
is missing or fails to load, importing this module raises -- there is no
eager/PyTorch/CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsinkattn.so")

# st_status codes (include/sinkattn.h)
ST_OK = 0
ST_INVALID_ARGUMENT = 1
ST_INFEASIBLE_SUPPORT = 2
ST_INVALID_TEMPERATURE = 3
ST_UNSUPPORTED_DEPTH = 4
ST_MISSING_BASE_TRACE = 5
ST_SIZE_CAP_EXCEEDED = 6
ST_CUDA_ERROR = 7
ST_WORKSPACE_TOO_SMALL = 8
ST_NOT_SUPPORTED = 9

ST_F32 = 0
ST_BF16 = 1
ST_FLAG_GENERIC = 1
ST_FLAG_REUSE_BAND = 2
ST_FLAG_STORED_BAND = 4
ST_MAX_STAGES = 8
ST_ONE_REFERENCE = 0
ST_DIRECT_FOUR_PLAN = 1
ST_GENERIC_TAIL = 2

# every symbol include/sinkattn.h declares
EXPORTED = (
    "st_saved_bytes", "st_workspace_bytes", "st_forward", "st_backward", "st_saved_duals",
    "st_validate_support", "st_normal_fill", "st_uniform_fill", "st_last_error", "st_launch_count",
    "st_forward_halo", "st_backward_halo", "st_base_vjp_workspace_bytes", "st_base_solve_vjp",
    "st_tail_adjoint", "st_check_status",
)


class StDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int64), ("heads", ctypes.c_int64), ("seq_q", ctypes.c_int64),
        ("seq_k", ctypes.c_int64), ("head_dim", ctypes.c_int64), ("half_band", ctypes.c_int64),
        ("base_depth", ctypes.c_int64), ("tail_depth", ctypes.c_int64), ("epsilon", ctypes.c_double),
        ("dtype", ctypes.c_int32), ("dustbin", ctypes.c_int32), ("dustbin_cost", ctypes.c_double),
        ("centered", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("n_stages", ctypes.c_int32), ("stage_eps", ctypes.POINTER(ctypes.c_double)),
        ("stage_iters", ctypes.POINTER(ctypes.c_int64)),
    ]


# void (*st_halo_fn)(void* user, int32_t kind, float* vec, int64_t len, void* stream)
HALO_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2605_08123_b200/csrc). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, VP, D, I64, I32, U64 = (ctypes.POINTER(StDesc), ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                               ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64)
    lib.st_saved_bytes.argtypes = [P]
    lib.st_saved_bytes.restype = ctypes.c_size_t
    lib.st_workspace_bytes.argtypes = [P]
    lib.st_workspace_bytes.restype = ctypes.c_size_t
    lib.st_forward.argtypes = [P, VP, VP, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP]
    lib.st_forward.restype = ctypes.c_int
    lib.st_backward.argtypes = [P, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, I32, VP, ctypes.c_size_t, VP]
    lib.st_backward.restype = ctypes.c_int
    lib.st_forward_halo.argtypes = [P, VP, VP, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP, HALO_FN, VP]
    lib.st_forward_halo.restype = ctypes.c_int
    lib.st_backward_halo.argtypes = [P, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, I32, VP, ctypes.c_size_t,
                                     VP, HALO_FN, VP, I64, I64]
    lib.st_backward_halo.restype = ctypes.c_int
    lib.st_tail_adjoint.argtypes = [P, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP]
    lib.st_tail_adjoint.restype = ctypes.c_int
    lib.st_base_vjp_workspace_bytes.argtypes = [P]
    lib.st_base_vjp_workspace_bytes.restype = ctypes.c_size_t
    lib.st_base_solve_vjp.argtypes = [P, VP, VP, VP, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP]
    lib.st_base_solve_vjp.restype = ctypes.c_int
    lib.st_saved_duals.argtypes = [P, VP, VP, VP, D, D, D, VP]
    lib.st_saved_duals.restype = ctypes.c_int
    lib.st_check_status.argtypes = [P, VP, VP]
    lib.st_check_status.restype = ctypes.c_int
    lib.st_validate_support.argtypes = [P, VP, VP]
    lib.st_validate_support.restype = ctypes.c_int
    lib.st_normal_fill.argtypes = [U64, ctypes.c_char_p, U64, I64, ctypes.c_double, D]
    lib.st_normal_fill.restype = None
    lib.st_uniform_fill.argtypes = [U64, ctypes.c_char_p, U64, I64, D]
    lib.st_uniform_fill.restype = None
    lib.st_last_error.argtypes = []
    lib.st_last_error.restype = ctypes.c_char_p
    lib.st_launch_count.argtypes = [I32]
    lib.st_launch_count.restype = I64
    return lib


lib = _load()
