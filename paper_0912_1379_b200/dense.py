"""Dense O(n^2) transforms on the GPU -- the reference's correctness oracles
(SURVEY 8(f) item 4), made matrix-free and fast.

Entry-by-entry evaluations of the closed-form matrices, independent of the fast
chirp-DFT-chirp / Bluestein kernels (no FFT, no chirp factorisation shared):

* ``scaled_fourier_matrix`` F = C(n) p_j e^{-2 pi i (jk mod n)/n} p_k   (xft/kernel.py:68-80)
* ``dense_lct_matrix``      L = S1 F S2                                  (xft/dense.py:230-249)
* ``frft_matrix_asymptotic`` entries K_z(x_j, x_k) dx                     (xft/dense.py:122-151)

``*_apply`` run matrix-free for any n (a full-size config-3 row, n = 16384,
takes milliseconds); ``*_entries`` materialise n <= 4096 (MAX_DENSE_N,
xft/dense.py:44), like the reference.  complex128 throughout.
"""
from __future__ import annotations

import numpy as np

from . import _native, ops
from .errors import DegenerateParameterError, InvalidSizeError, ShapeError

MAX_DENSE_N = 4096  # xft/dense.py:44

KIND_F, KIND_LCT, KIND_MEHLER = 0, 1, 2

__all__ = ["MAX_DENSE_N", "dense_lct_apply", "dense_mehler_apply", "dense_entries", "dense_lct_matrix",
           "scaled_fourier_matrix_gpu"]


def _rows128(values):
    """[B, n] complex128 CUDA tensor view of ``values`` (numpy or torch; a 1-D vector is one row)."""
    torch = ops._torch()
    if isinstance(values, np.ndarray):
        values = torch.from_numpy(np.ascontiguousarray(values, dtype=np.complex128)).cuda()
    v = values if values.ndim == 2 else values.reshape(1, -1)
    if v.dtype != torch.complex128:
        v = v.to(torch.complex128)
    return v.contiguous()


def _check_dense_size(n: int) -> None:
    if isinstance(n, bool) or not isinstance(n, (int, np.integer)) or n < 1:
        raise InvalidSizeError(f"size must be a positive integer, got {n!r}")
    if n > MAX_DENSE_N:
        raise InvalidSizeError(f"dense path materializes only n <= {MAX_DENSE_N} (got {n})")


def dense_lct_apply(values, abcd=None, *, out=None):
    """L @ v for every row (abcd None: F @ v), O(n^2) on the GPU, no matrix stored."""
    torch = ops._torch()
    v = _rows128(values)
    B, n = v.shape
    p = None
    if abcd is not None:
        p = np.ascontiguousarray(np.asarray(abcd, dtype=np.float64).reshape(4))
        if p[1] == 0:
            raise DegenerateParameterError("b = 0 has no kernel matrix; use lct_b_zero")
    out = ops.check_out(out, v)
    with torch.cuda.device(v.device):
        _native.call("xft_dense_lct_apply", v.data_ptr(), out.data_ptr(), B, n,
                     None if p is None else p.ctypes.data, ops._stream_ptr(v.device))
    return out


def dense_mehler_apply(values, z, *, out=None):
    """(K_z(x_j, x_k) dx) @ f for every row, O(n^2) on the GPU; z: one order or one per row."""
    from .mehler import _check_z

    torch = ops._torch()
    v = _rows128(values)
    B, n = v.shape
    zz = _check_z(z)
    if zz.shape[0] not in (1, B):
        raise ShapeError(f"{zz.shape[0]} orders for a batch of {B}")
    zh = np.ascontiguousarray(np.stack([zz.real, zz.imag], axis=1))
    out = ops.check_out(out, v)
    with torch.cuda.device(v.device):
        _native.call("xft_dense_mehler_apply", v.data_ptr(), out.data_ptr(), B, n, zh.ctypes.data,
                     0 if zh.shape[0] == 1 else 2, ops._stream_ptr(v.device))
    return out


def dense_entries(n: int, kind: int, param=None):
    """[n, n] complex128 CUDA tensor of F (kind 0), L (1, param = abcd) or K_z dx (2, param = z)."""
    torch = ops._torch()
    _check_dense_size(n)
    if kind == KIND_MEHLER:
        z = complex(param)
        ph = np.array([z.real, z.imag], dtype=np.float64)
    elif kind == KIND_LCT:
        ph = np.ascontiguousarray(np.asarray(param, dtype=np.float64).reshape(4))
        if ph[1] == 0:
            raise DegenerateParameterError("b = 0 has no kernel matrix; use lct_b_zero")
    else:
        ph = None
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((n, n), dtype=torch.complex128, device=dev)
    _native.call("xft_dense_entries", out.data_ptr(), n, int(kind), None if ph is None else ph.ctypes.data,
                 ops._stream_ptr(dev))
    return out


def scaled_fourier_matrix_gpu(n: int) -> np.ndarray:
    """F (xft/kernel.py:68-80) built on the GPU, returned as numpy."""
    return dense_entries(n, KIND_F).cpu().numpy()


def dense_lct_matrix(n: int, params):
    """Materialised LCT matrix L = S1 F S2 on the asymptotic grid (reference: xft/dense.py:230-249)."""
    from .mehler import DenseTransform

    _check_dense_size(n)
    if params.b == 0:
        raise DegenerateParameterError("b = 0 has no kernel matrix; use lct_b_zero")
    return DenseTransform(n=int(n), provenance="lct", detail=params.as_tuple())
