"""DFT plans and application (drop-in for xft.fftcore), GPU-backed.

Semantics (reference: xft/fftcore.py:1-19): out[j] = sum_k e^{s 2 pi i jk/n} v[k],
unnormalised, any n >= 1.  A plan is immutable, owns no scratch and may be
shared between host threads (xft/fftcore.py:8-11): on the device it is the
lazily built twiddle table of libxft_b200.so (``xft_prepare``), keyed by
(device, n, dtype).  Route selection mirrors the reference
(xft/fftcore.py:80-100): "radix-2" for powers of two, "chirp-z" (Bluestein
into a power-of-two convolution, executed inside one kernel) otherwise.
"""
from __future__ import annotations

import numpy as np

from . import ops
from .errors import InvalidSizeError, ParameterError, ShapeError

__all__ = ["DftPlan", "plan_dft", "apply_dft", "naive_dft"]

NAIVE_CAP = 4096  # xft/fftcore.py:21


class DftPlan:
    """Reusable plan for one (length, direction) pair (reference: xft/fftcore.py:57-100)."""

    __slots__ = ("n", "direction_sign", "route", "_m")

    def __init__(self, n: int, direction_sign: int):
        if isinstance(n, bool) or not isinstance(n, (int, np.integer)) or n < 1:
            raise InvalidSizeError(f"transform length must be positive, got {n!r}")
        if direction_sign not in (1, -1):
            raise ParameterError(f"direction_sign must be +1 or -1, got {direction_sign!r}")
        self.n = int(n)
        self.direction_sign = int(direction_sign)
        if self.n & (self.n - 1) == 0:
            self.route = "radix-2"
            self._m = self.n
        else:
            self.route = "chirp-z"
            m = 1
            while m < 2 * self.n - 1:
                m *= 2
            self._m = m


def plan_dft(n: int, direction_sign: int) -> DftPlan:
    """Create a plan (reference: xft/fftcore.py:103-105)."""
    return DftPlan(n, direction_sign)


def apply_dft(plan: DftPlan, v) -> np.ndarray:
    """Apply a plan to a length-n vector; returns a fresh complex128 array (xft/fftcore.py:108-119)."""
    v = np.asarray(v)
    if v.ndim != 1 or v.shape[0] != plan.n:
        raise ShapeError(f"expected a vector of length {plan.n}, got shape {v.shape}")
    torch = ops._torch()
    t = torch.from_numpy(v.astype(complex, copy=True)).to("cuda")
    out = ops.dft_rows(t, plan.direction_sign)
    return out[0].cpu().numpy()


def apply_dft_batch(plan: DftPlan, values):
    """Batched device variant: ``values`` [B, n] complex CUDA tensor -> CUDA tensor."""
    if values.shape[-1] != plan.n:
        raise ShapeError(f"expected rows of length {plan.n}, got {tuple(values.shape)}")
    return ops.dft_rows(values, plan.direction_sign)


def naive_dft(v, direction_sign: int) -> np.ndarray:
    """Quadratic-time DFT oracle (reference: xft/fftcore.py:122-137), on the GPU.

    out[j] = sum_k exp(sign 2 pi i ((j k) mod n) / n) v[k], evaluated entry by
    entry (``xft_naive_dft``: no FFT, shares nothing with the fast path), same
    checks and order as the reference: sign, empty input, the n <= 4096 cap.
    """
    from . import _native

    if direction_sign not in (1, -1):
        raise ParameterError(f"direction_sign must be +1 or -1, got {direction_sign!r}")
    v = np.asarray(v, dtype=complex)
    n = v.shape[0]
    if n < 1:
        raise InvalidSizeError("empty input")
    if n > NAIVE_CAP:
        raise InvalidSizeError(f"naive DFT capped at n={NAIVE_CAP} (got {n})")
    torch = ops._torch()
    t = ops.aligned(torch.from_numpy(np.ascontiguousarray(v.reshape(1, n))).to("cuda"))
    out = torch.empty_like(t)
    with torch.cuda.device(t.device):
        _native.call("xft_naive_dft", t.data_ptr(), out.data_ptr(), 1, n, int(direction_sign),
                     ops._stream_ptr(t.device))
    return out[0].cpu().numpy()
