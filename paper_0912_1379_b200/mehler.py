"""Complex-z fractional Fourier transform (Mehler kernel), GPU-backed.

Semantics of the reference's frft_matrix_asymptotic (xft/dense.py:139-151):
g_j = sum_k K_z(x_j, x_k) dx f_k on the asymptotic grid, with
K_z(x,y) = sqrt(2/(1-z^2)) exp(-((1+z^2)(x^2+y^2) - 4xyz) / (2(1-z^2)))
(xft/dense.py:122-136).  The reference materialises the n x n matrix (n <= 4096);
here ``apply`` runs the O(n log n) windowed Bluestein kernel of libxft_b200.so
for any n, and the dense ``entries`` are only built on request (n <= 4096, on
the GPU, entry by entry -- see dense.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native, ops
from .errors import InvalidSizeError, ParameterError, ShapeError, SingularParameterError
from .hermite import asymptotic_zeros

MAX_DENSE_N = 4096            # xft/dense.py:44
_UNIT_DISK_TOL = 1e-12        # xft/dense.py:45
_SINGULAR_TOL = 1e-14         # xft/dense.py:46


@dataclass(frozen=True)
class FrftOrder:
    """Complex order z, |z| <= 1 (reference: xft/dense.py:49-59)."""

    z: complex

    def __post_init__(self):
        z = complex(self.z)
        if abs(z) > 1.0 + _UNIT_DISK_TOL:
            raise ParameterError(f"|z| = {abs(z)!r} lies outside the closed unit disk")
        object.__setattr__(self, "z", z)


def mehler_kernel(order: FrftOrder, x, y):
    """K_z(x, y), principal sqrt branch (reference: xft/dense.py:122-136); host helper."""
    z = complex(order.z)
    if abs(z - 1.0) < _SINGULAR_TOL or abs(z + 1.0) < _SINGULAR_TOL:
        raise SingularParameterError(f"kernel is singular at z = {z} (1 - z^2 = 0)")
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    one = 1.0 - z * z
    expo = -((1.0 + z * z) * (x * x + y * y) - 4.0 * x * y * z) / (2.0 * one)
    out = np.sqrt(2.0 / one) * np.exp(expo)
    return complex(out) if out.ndim == 0 else out


def _check_z(z) -> np.ndarray:
    zz = np.asarray(z, dtype=complex).reshape(-1)
    for v in zz:
        FrftOrder(v)
        if abs(v - 1.0) < _SINGULAR_TOL or abs(v + 1.0) < _SINGULAR_TOL:
            raise SingularParameterError(f"kernel is singular at z = {v} (1 - z^2 = 0)")
    return zz


def mehler_rows(values, z, *, out=None):
    """Batched Mehler transform of the rows of ``values`` ([B, n] complex128 CUDA tensor).

    ``z``: one complex order for all rows, or B of them (host values).
    """
    torch = ops._torch()
    v = ops._rows_view(values)
    if v.dtype != torch.complex128:
        raise ParameterError("the Mehler transform runs in complex128 (1e-12 tolerance)")
    B, n = v.shape
    zz = _check_z(z)
    if zz.shape[0] not in (1, B):
        raise ShapeError(f"{zz.shape[0]} orders for a batch of {B}")
    zh = np.ascontiguousarray(np.stack([zz.real, zz.imag], axis=1))
    out = ops.check_out(out, v)
    with torch.cuda.device(v.device):
        _native.call("xft_mehler", v.data_ptr(), out.data_ptr(), B, n, zh.ctypes.data,
                     0 if zh.shape[0] == 1 else 2, None, ops._stream_ptr(v.device))
    return out


class MehlerPlan:
    """Caller-owned device plan for one z array (``xft_mehler_plan_create``).

    The per-row parameters, size classes and row lists that ``mehler_rows``
    otherwise takes from the library's implicit cache, held by the caller: a
    CUDA graph captured around ``apply`` stays valid for as long as the plan
    object lives, whatever else the process transforms.  Immutable; ``apply``
    may run from several threads/streams at once.  ``close()`` (or garbage
    collection) frees it -- only after the work and graphs using it are done.
    """

    def __init__(self, n: int, z, device=None):
        import ctypes

        torch = ops._torch()
        zz = _check_z(z)
        self.n, self.batch = int(n), int(zz.shape[0])
        if self.n < 1:
            raise InvalidSizeError(f"transform length must be positive, got {n!r}")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        zh = np.ascontiguousarray(np.stack([zz.real, zz.imag], axis=1))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.call("xft_mehler_plan_create", self.batch, self.n, zh.ctypes.data, 2, ctypes.byref(h))
        self._h = h.value

    def apply(self, values, *, out=None):
        torch = ops._torch()
        if self._h is None:
            raise ParameterError("the plan has been closed")
        v = ops._rows_view(values)
        if v.dtype != torch.complex128:
            raise ParameterError("the Mehler transform runs in complex128 (1e-12 tolerance)")
        if tuple(v.shape) != (self.batch, self.n):
            raise ShapeError(f"plan is for [{self.batch}, {self.n}], got {tuple(v.shape)}")
        if v.device != self.device:
            raise ShapeError(f"plan lives on {self.device}, values on {v.device}")
        out = ops.check_out(out, v)
        with torch.cuda.device(v.device):
            _native.call("xft_mehler_planned", v.data_ptr(), out.data_ptr(), self._h, None,
                         ops._stream_ptr(v.device))
        return out

    def close(self):
        if getattr(self, "_h", None) is not None:
            _native.lib().xft_mehler_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def release_caches():
    """Frees the implicit plan cache, retired plans and internal scratch (``xft_release_caches``).

    Call only when no queued work or live CUDA graph uses them."""
    _native.call("xft_release_caches")


@dataclass(frozen=True)
class DenseTransform:
    """Drop-in for the reference's DenseTransform (xft/dense.py:62-80).

    provenance "chirp_factored" (frft_matrix_asymptotic, detail = z) or "lct"
    (dense_lct_matrix, detail = (a, b, c, d)).  ``entries`` are built on the GPU
    entry by entry (n <= 4096); ``apply`` runs the fast kernel for the Mehler
    case and the matrix-free dense product for "lct"; ``apply_dense`` is always
    the O(n^2) entry-by-entry product (any n) -- the independent check.
    """

    n: int
    provenance: str
    detail: object = field(default=None)

    def _kind(self):
        from . import dense

        return dense.KIND_MEHLER if self.provenance == "chirp_factored" else dense.KIND_LCT

    @property
    def entries(self) -> np.ndarray:
        from . import dense

        if self.n > MAX_DENSE_N:
            raise InvalidSizeError(f"dense path materializes only n <= {MAX_DENSE_N} (got {self.n})")
        return dense.dense_entries(self.n, self._kind(), self.detail).cpu().numpy()

    def _vector(self, v):
        v = np.asarray(v, dtype=complex)
        if v.shape != (self.n,):
            raise ShapeError(f"expected a vector of length {self.n}, got {v.shape}")
        return v

    def apply(self, v) -> np.ndarray:
        v = self._vector(v)
        if self.provenance != "chirp_factored":
            return self.apply_dense(v)
        torch = ops._torch()
        t = torch.from_numpy(v).to("cuda")
        return mehler_rows(t, self.detail)[0].cpu().numpy()

    def apply_dense(self, v) -> np.ndarray:
        from . import dense

        v = self._vector(v)
        if self.provenance == "chirp_factored":
            return dense.dense_mehler_apply(v, self.detail)[0].cpu().numpy()
        return dense.dense_lct_apply(v, self.detail)[0].cpu().numpy()


def frft_matrix_asymptotic(n: int, order: FrftOrder) -> DenseTransform:
    """K_z(x_j, x_k) dx on the asymptotic grid (reference: xft/dense.py:139-151); fast ``apply``."""
    if isinstance(n, bool) or not isinstance(n, (int, np.integer)) or n < 1:
        raise InvalidSizeError(f"size must be a positive integer, got {n!r}")
    z = complex(order.z)
    if abs(z - 1.0) < _SINGULAR_TOL or abs(z + 1.0) < _SINGULAR_TOL:
        raise SingularParameterError(f"kernel is singular at z = {z} (1 - z^2 = 0)")
    return DenseTransform(n=int(n), provenance="chirp_factored", detail=z)


def fast_mehler_frft(order: FrftOrder, signal) -> np.ndarray:
    """g = frft_matrix_asymptotic(n, order).apply(signal.values) without the dense matrix."""
    return frft_matrix_asymptotic(signal.grid.n, order).apply(signal.values)
