"""ctypes binding of the C-ABI library ``libxft_b200.so`` (include/xft_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every
transform raises ``NativeUnavailable`` -- the package never computes a
transform on the CPU.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import XftError, raise_for

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libxft_b200.so")

C64 = 0
C128 = 1
FLAG_BARE_FOURIER = 1


class NativeUnavailable(XftError, RuntimeError):
    """The CUDA library or device is unavailable (no CPU fallback exists)."""


_lock = threading.Lock()
_lib = None

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "xft_version": ([], ctypes.c_int),
    "xft_max_n": ([ctypes.c_int], _i64),
    "xft_prepare": ([_i64, ctypes.c_int], ctypes.c_int),
    "xft_validate_lct_params": ([_vp, _i64, _i64, ctypes.c_int, ctypes.c_double, ctypes.POINTER(_i64)], ctypes.c_int),
    "xft_lct": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, ctypes.c_int, _vp], ctypes.c_int),
    "xft_lct_checked": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "xft_dft": ([_vp, _vp, _i64, _i64, ctypes.c_int, ctypes.c_int, _vp], ctypes.c_int),
    "xft_scaled_fourier": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp], ctypes.c_int),
    "xft_lct_host": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_double],
                     ctypes.c_int),
    "xft_mehler_workspace_bytes": ([_i64, _i64], _i64),
    "xft_mehler": ([_vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp], ctypes.c_int),
    "xft_validate_mehler_z": ([_vp, _i64, _i64, ctypes.POINTER(_i64)], ctypes.c_int),
    "xft_mehler_plan_create": ([_i64, _i64, _vp, _i64, ctypes.POINTER(_vp)], ctypes.c_int),
    "xft_mehler_planned": ([_vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "xft_mehler_plan_destroy": ([_vp], ctypes.c_int),
    "xft_release_caches": ([], ctypes.c_int),
    "xft_lct2d": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp], ctypes.c_int),
    "xft_lct2d_sharded": ([_vp, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "xft_nccl_info": ([ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "xft_transpose": ([_vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp], ctypes.c_int),
    "xft_lct_columns": ([_vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp], ctypes.c_int),
    "xft_column_schedule": ([_i64, _i64, _i64, _vp, _vp], ctypes.c_int),
    "xft_lct_rows_packed": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, ctypes.c_int, _i64, _vp], ctypes.c_int),
    "xft_lct_rows_peers": ([_vp, _vp, ctypes.c_int, _i64, _i64, _i64, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "xft_lct_chain": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, _vp],
                      ctypes.c_int),
    "xft_lct_b_zero": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _vp], ctypes.c_int),
    "xft_validate_b_zero": ([_vp, _i64, _i64, ctypes.c_double, ctypes.POINTER(_i64)], ctypes.c_int),
    "xft_dense_lct_apply": ([_vp, _vp, _i64, _i64, _vp, _vp], ctypes.c_int),
    "xft_dense_mehler_apply": ([_vp, _vp, _i64, _i64, _vp, _i64, _vp], ctypes.c_int),
    "xft_naive_dft": ([_vp, _vp, _i64, _i64, ctypes.c_int, _vp], ctypes.c_int),
    "xft_dense_entries": ([_vp, _i64, ctypes.c_int, _vp, _vp], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no device needed)."""
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = load_library()
    return _lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise the mapped exception."""
    status = getattr(lib(), name)(*args)
    raise_for(status, name)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the XFT transforms run only on the GPU")
    return torch
