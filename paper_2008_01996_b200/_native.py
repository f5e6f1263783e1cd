"""ctypes binding of libkhb200.so (the C-ABI in include/khb200.h).

The library is built in-tree by `build.py` (nvcc, sm_100a). There is no CPU
fallback: if the library is missing or no CUDA device is present, every
entry point that needs it raises `DeviceError`.
"""

import ctypes
import os

from .errors import DeviceError, DimensionMismatch, SingularMatrix, UsageError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkhb200.so")
# instrumented / experimental builds of the same sources (profiles/probes) can be
# loaded instead for measurements; the product path uses the in-tree library
if os.environ.get("KHB200_LIB"):
    LIB_PATH = os.environ["KHB200_LIB"]

KH_OK = 0
KH_ERR_DIMENSION = 1
KH_ERR_SINGULAR = 2
KH_ERR_INVALID = 3
KH_ERR_CUDA = 4
KH_ERR_NOMEM = 5

_STATUS_EXC = {
    KH_ERR_DIMENSION: DimensionMismatch,
    KH_ERR_SINGULAR: SingularMatrix,
    KH_ERR_INVALID: UsageError,
    KH_ERR_CUDA: DeviceError,
    KH_ERR_NOMEM: DeviceError,
}


class SymbolicStats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("n_fronts", ctypes.c_int64),
        ("max_front", ctypes.c_int64),
        ("max_pivots", ctypes.c_int64),
        ("depth", ctypes.c_int64),
        ("factor_nnz", ctypes.c_int64),
        ("panel_entries", ctypes.c_int64),
        ("upd_entries", ctypes.c_int64),
        ("leaf_size", ctypes.c_int64),
        ("flops", ctypes.c_double),
    ]


_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_P = ctypes.POINTER

# name -> (restype, argtypes); every symbol include/khb200.h declares
SIGNATURES = {
    "kh_version": (ctypes.c_int, []),
    "kh_launch_count": (ctypes.c_int64, []),
    "kh_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "kh_last_error": (ctypes.c_char_p, []),
    "kh_analyze": (ctypes.c_int, [_i64, _vp, _vp, _i32, _P(_vp)]),
    "kh_analyze_union": (ctypes.c_int, [_i64, _vp, _vp, _vp, _vp, _i32, _P(_vp)]),
    "kh_symbolic_stats_get": (ctypes.c_int, [_vp, _P(SymbolicStats)]),
    "kh_symbolic_perm": (ctypes.c_int, [_vp, _vp]),
    "kh_symbolic_fronts": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "kh_symbolic_rows": (ctypes.c_int, [_vp, _vp]),
    "kh_symbolic_pattern": (ctypes.c_int, [_vp, _vp, _vp]),
    "kh_align_values": (ctypes.c_int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kh_symbolic_free": (None, [_vp]),
    "kh_plan_create": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _i64, _P(_vp)]),
    "kh_plan_bytes": (ctypes.c_int, [_vp, _i64, _i64, _P(_i64)]),
    "kh_plan_set_values": (ctypes.c_int, [_vp, _vp, _vp]),
    "kh_plan_factor": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "kh_plan_pivot_check": (ctypes.c_int, [_vp, _i64, _i64, _dbl, _vp, _P(_i64), _P(_dbl)]),
    "kh_plan_solve": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp]),
    "kh_plan_factor_solve": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _vp]),
    "kh_plan_factor_fwd": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _i64, _vp]),
    "kh_plan_solve_bwd": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _i64, _vp]),
    "kh_plan_factor_storage": (ctypes.c_int, [_vp, _P(_vp), _P(_i64)]),
    "kh_plan_set_level_timing": (ctypes.c_int, [_vp, _i32]),
    "kh_plan_level_times": (ctypes.c_int, [_vp, _vp, _i32]),
    "kh_plan_residual": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "kh_plan_residual_scale": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "kh_plan_residual_dd": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "kh_dgemm_dd": (ctypes.c_int, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp]),
    "kh_csr_pair_residual_dd": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64,
                                               _vp, _i64, _vp, _vp]),
    "kh_plan_free": (None, [_vp]),
    "kh_dgemm": (ctypes.c_int, [_i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp]),
    "kh_sumsq": (ctypes.c_int, [_vp, _i64, _vp, _vp]),
    "kh_daxpy": (ctypes.c_int, [_i64, _dbl, _vp, _vp, _vp]),
    "kh_csr_pair_residual": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                                            _vp, _vp]),
    "kh_dgemm_rowscatter": (ctypes.c_int, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i32, _i64, _i64, _vp]),
    "kh_sum_parts": (ctypes.c_int, [_i32, _vp, _i64, _vp, _vp]),
    "kh_ipc_handle": (ctypes.c_int, [_vp, _vp, _P(_i64)]),
    "kh_ipc_open": (ctypes.c_int, [_vp, _P(_vp)]),
    "kh_ipc_close": (ctypes.c_int, [_vp]),
    "kh_ht_workspace_bytes": (ctypes.c_int, [_i32, _i64, _P(_i64)]),
    "kh_ht_assemble": (ctypes.c_int, [_i32, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "kh_set_device": (ctypes.c_int, [ctypes.c_int]),
    "kh_stream_sync": (ctypes.c_int, [_vp]),
}

_lib = None


def load():
    """Load libkhb200.so (raises DeviceError if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status):
    if status == KH_OK:
        return
    lib = load()
    msg = lib.kh_last_error().decode(errors="replace")
    exc = _STATUS_EXC.get(status, DeviceError)
    raise exc(msg or lib.kh_status_string(status).decode())


def call(name, *args):
    check(getattr(load(), name)(*args))


def ptr(t):
    """Raw pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def launch_count():
    """Kernel launches made by libkhb200 so far (for bench.py's gpu_launches)."""
    return int(load().kh_launch_count())


def require_cuda():
    """The product path runs only on a CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available; the B200 solver has no CPU fallback")
    load()


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
