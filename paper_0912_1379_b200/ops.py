"""Device-level batched operators: torch CUDA tensors in, torch CUDA tensors out.

Each function is a thin shim over one C-ABI entry point (include/xft_b200.h):
it checks shapes/dtypes, allocates the output, and launches on the current
torch stream.  torch is only the allocator / stream provider here; all
arithmetic runs in the hand-written sm_100a kernels of libxft_b200.so.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import InvalidSizeError, ParameterError, ShapeError

UNIMODULAR_TOL = 1e-10


def _torch():
    return _native.require_cuda()


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.complex64:
        return _native.C64
    if t.dtype == torch.complex128:
        return _native.C128
    raise ParameterError(f"complex64 or complex128 required, got {t.dtype}")


def _stream_ptr(device) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


ALIGN = 16  # bytes: rows move with cp.async.bulk (include/xft_b200.h "Alignment")


def aligned(t):
    """``t`` contiguous and 16-byte aligned (a copy when the view is not)."""
    t = t.contiguous()
    if t.numel() and t.data_ptr() % ALIGN:
        t = t.clone()  # fresh allocations are 256-byte aligned
    return t


def _rows_view(values, what="values"):
    if values.dim() == 1:
        values = values.unsqueeze(0)
    if values.dim() != 2:
        raise ShapeError(f"{what} must be [batch, n], got shape {tuple(values.shape)}")
    if values.shape[1] < 1:
        raise InvalidSizeError(f"transform length must be positive, got {values.shape[1]}")
    if not values.is_cuda:
        raise ShapeError(f"{what} must be a CUDA tensor")
    return aligned(values)


def check_out(out, like, shape=None):
    """A caller-supplied ``out`` must match exactly: shape, dtype, device, contiguous, 16-byte aligned.

    (The kernels write through the raw pointer; a wrong ``out`` would be an
    out-of-bounds device write.)  Returns ``out``; allocates when it is None."""
    torch = _torch()
    shape = tuple(like.shape) if shape is None else tuple(shape)
    if out is None:
        return torch.empty(shape, dtype=like.dtype, device=like.device)
    if not isinstance(out, torch.Tensor):
        raise ShapeError(f"out must be a torch tensor, got {type(out).__name__}")
    if tuple(out.shape) != shape:
        raise ShapeError(f"out has shape {tuple(out.shape)}, expected {shape}")
    if out.dtype != like.dtype:
        raise ParameterError(f"out has dtype {out.dtype}, expected {like.dtype}")
    if out.device != like.device:
        raise ShapeError(f"out is on {out.device}, expected {like.device}")
    if not out.is_contiguous():
        raise ShapeError("out must be contiguous")
    if out.numel() and out.data_ptr() % ALIGN:
        raise ShapeError(f"out must be {ALIGN}-byte aligned")
    return out


def check_out_host(out, like: np.ndarray):
    """Host-buffer variant of ``check_out`` for numpy arrays."""
    if out is None:
        return np.empty_like(like)
    if not isinstance(out, np.ndarray):
        raise ShapeError(f"out must be a numpy array, got {type(out).__name__}")
    if out.shape != like.shape:
        raise ShapeError(f"out has shape {out.shape}, expected {like.shape}")
    if out.dtype != like.dtype:
        raise ParameterError(f"out has dtype {out.dtype}, expected {like.dtype}")
    if not out.flags.c_contiguous or not out.flags.writeable:
        raise ShapeError("out must be a writeable C-contiguous array")
    return out


def validate_abcd_host(abcd: np.ndarray, check_unimodular=True, tol=UNIMODULAR_TOL) -> None:
    """Reference-order validation (b == 0 first, then unimodularity) on a host copy."""
    a = np.ascontiguousarray(abcd, dtype=np.float64)
    rows = a.reshape(-1, 4)
    bad = ctypes.c_int64(-1)
    status = _native.lib().xft_validate_lct_params(
        a.ctypes.data, rows.shape[0], 4 if rows.shape[0] > 1 or a.ndim == 2 else 0,
        int(bool(check_unimodular)), float(tol), ctypes.byref(bad))
    if status:
        from .errors import raise_for
        raise_for(status, f"LCT parameters (row {bad.value})")


def lct_rows(values, abcd, *, bare_fourier=False, out=None, validate=True,
             check_unimodular=True, tol=UNIMODULAR_TOL, check_finite=False):
    """Batched fast LCT of the rows of ``values`` ([B, n] complex64/complex128, CUDA).

    ``abcd``: 4 numbers (one quadruple for every row), a [B, 4] array, or a
    [B, 4] float64 CUDA tensor (per-row parameters, e.g. FrFT angles).
    Reference semantics: fast_lct (xft/lct.py:168-208) applied to every row.
    ``check_finite``: the reference's Signal check (xft/lct.py:125-126) for the
    whole batch, fused into the row kernel (``xft_lct_checked``); raises
    ParameterError naming the first non-finite row (this synchronises the stream).
    """
    torch = _torch()
    v = _rows_view(values)
    B, n = v.shape
    if isinstance(abcd, torch.Tensor) and abcd.is_cuda:
        p_dev = abcd.to(torch.float64).reshape(-1, 4).contiguous()
        if validate:
            validate_abcd_host(p_dev.cpu().numpy(), check_unimodular, tol)
    else:
        p_host = np.ascontiguousarray(np.asarray(abcd, dtype=np.float64).reshape(-1, 4))
        if validate:
            validate_abcd_host(p_host, check_unimodular, tol)
        p_dev = torch.from_numpy(p_host).to(v.device, non_blocking=False)
    if p_dev.shape[0] not in (1, B):
        raise ShapeError(f"abcd has {p_dev.shape[0]} rows for a batch of {B}")
    stride = 0 if p_dev.shape[0] == 1 else 4
    out = check_out(out, v)
    flags = _native.FLAG_BARE_FOURIER if bare_fourier else 0
    with torch.cuda.device(v.device):
        if check_finite:
            bad = torch.empty(1, dtype=torch.int64, device=v.device)
            _native.call("xft_lct_checked", v.data_ptr(), out.data_ptr(), B, n, _dtype_code(v),
                         p_dev.data_ptr(), stride, flags, bad.data_ptr(), _stream_ptr(v.device))
            first = int(bad.item())
            if first < B:
                raise ParameterError(f"signal values must be finite (row {first})")
        else:
            _native.call("xft_lct", v.data_ptr(), out.data_ptr(), B, n, _dtype_code(v),
                         p_dev.data_ptr(), stride, flags, _stream_ptr(v.device))
    # p_dev may be released now: the caching allocator only reuses its block
    # in order on this same stream.
    return out


def dft_rows(values, sign: int, *, out=None):
    """Batched unnormalised DFT (apply_dft, xft/fftcore.py:108-119) of every row."""
    torch = _torch()
    if sign not in (1, -1):
        raise ParameterError(f"direction_sign must be +1 or -1, got {sign!r}")
    v = _rows_view(values)
    B, n = v.shape
    out = check_out(out, v)
    with torch.cuda.device(v.device):
        _native.call("xft_dft", v.data_ptr(), out.data_ptr(), B, n, int(sign), _dtype_code(v),
                     _stream_ptr(v.device))
    return out


def scaled_fourier_rows(values, *, out=None):
    """Batched F v = C(n) p DFT(p v) (apply_scaled_fourier, xft/kernel.py:83-95)."""
    torch = _torch()
    v = _rows_view(values)
    B, n = v.shape
    out = check_out(out, v)
    with torch.cuda.device(v.device):
        _native.call("xft_scaled_fourier", v.data_ptr(), out.data_ptr(), B, n, _dtype_code(v),
                     _stream_ptr(v.device))
    return out


def transpose(values, *, out=None):
    """out = values.T (tiled device transpose used by the 2-D pass)."""
    torch = _torch()
    if values.dim() != 2 or not values.is_cuda:
        raise ShapeError("transpose needs a 2-D CUDA tensor")
    v = aligned(values)
    r, c = v.shape
    out = check_out(out, v, (c, r))
    with torch.cuda.device(v.device):
        _native.call("xft_transpose", v.data_ptr(), out.data_ptr(), r, c, c, r, _dtype_code(v),
                     _stream_ptr(v.device))
    return out


def lct_host(values: np.ndarray, abcd, *, bare_fourier=False, out=None,
             check_unimodular=True, tol=UNIMODULAR_TOL) -> np.ndarray:
    """End-to-end LCT on HOST arrays through ``xft_lct_host`` (chunked H2D/kernel/D2H pipeline).

    ``values``: [B, n] complex64/complex128 numpy array (pinned memory gives
    full link bandwidth).  Returns a numpy array of the same dtype.
    """
    _torch()
    v = np.ascontiguousarray(values)
    if v.ndim == 1:
        v = v[None, :]
    if v.dtype == np.complex64:
        code = _native.C64
    elif v.dtype == np.complex128:
        code = _native.C128
    else:
        raise ParameterError(f"complex64 or complex128 required, got {v.dtype}")
    p = np.ascontiguousarray(np.asarray(abcd, dtype=np.float64).reshape(-1, 4))
    if p.shape[0] not in (1, v.shape[0]):
        raise ShapeError(f"abcd has {p.shape[0]} rows for a batch of {v.shape[0]}")
    if v.ctypes.data % ALIGN:
        v = v.copy()  # numpy allocations are 16-byte aligned; a misaligned view is copied
    res = check_out_host(None if out is None else (out[None, :] if out.ndim == 1 else out), v)
    dst = res if res.ctypes.data % ALIGN == 0 else np.empty_like(v)
    flags = _native.FLAG_BARE_FOURIER if bare_fourier else 0
    _native.call("xft_lct_host", v.ctypes.data, dst.ctypes.data, v.shape[0], v.shape[1], code,
                 p.ctypes.data, 0 if p.shape[0] == 1 else 4, flags, int(bool(check_unimodular)), float(tol))
    if dst is not res:
        res[...] = dst
    return res if out is None or out.ndim != 1 else out


def lct_chain_rows(values, stages, *, scale=1.0, reverse=False, out=None):
    """L_k ... L_1 applied to every row in one launch (rows stay on chip between stages).

    ``stages``: sequence of (a, b, c, d); each stage reads the previous output as
    samples on the standard grid (xft/cli.py:236-253 semantics).
    """
    torch = _torch()
    v = _rows_view(values)
    B, n = v.shape
    p = np.ascontiguousarray(np.asarray(stages, dtype=np.float64).reshape(-1, 4))
    out = check_out(out, v)
    if B == 0:
        return out
    if not 1 <= p.shape[0] <= 4:
        raise ParameterError(f"a chain holds 1 to 4 stages (got {p.shape[0]})")
    if n & (n - 1) == 0 and 32 <= n <= (16384 if v.dtype == torch.complex64 else 8192):
        with torch.cuda.device(v.device):
            _native.call("xft_lct_chain", v.data_ptr(), out.data_ptr(), B, n, _dtype_code(v), p.ctypes.data,
                         p.shape[0], float(scale), int(bool(reverse)), _stream_ptr(v.device))
        return out
    # rows the one-launch chain does not hold on chip (non-powers of two, long or
    # short rows): the stages one after another through the row kernels
    cur = v
    for st in p:
        cur = lct_rows(cur, tuple(float(t) for t in st))
    if reverse:
        cur = cur.flip(1)
    out.copy_(cur * scale if scale != 1.0 else cur)
    return out


def inverse_roundtrip_rows(values, abcd, *, out=None):
    """Forward LCT then the scale-adjusted inverse (the reference CLI's --inverse, xft/cli.py:236-253).

    Recovers the input samples up to the discretisation error, in one launch.
    """
    import math

    a, b, c, d = (float(t) for t in np.asarray(abcd, dtype=np.float64).reshape(4))
    if b <= 0:
        raise ParameterError("--inverse requires b > 0")
    sigma = 4.0 * b / math.pi
    second = (d * sigma, -b / sigma, -c * sigma, a / sigma)
    return lct_chain_rows(values, [(a, b, c, d), second], scale=math.sqrt(sigma), reverse=True, out=out)


def lct_b_zero_rows(samples, abcd, *, out=None, tol=UNIMODULAR_TOL):
    """b = 0 branch for a batch: sqrt(d) e^{i c d y^2/2} f(d y) (xft/lct.py:236-263).

    ``samples``: [B, n] CUDA tensor of f(d y_j) values; ``abcd``: one quadruple or [B, 4].
    """
    torch = _torch()
    v = _rows_view(samples)
    B, n = v.shape
    p_host = np.ascontiguousarray(np.asarray(abcd, dtype=np.float64).reshape(-1, 4))
    bad = ctypes.c_int64(-1)
    st = _native.lib().xft_validate_b_zero(p_host.ctypes.data, p_host.shape[0], 4 if p_host.shape[0] > 1 else 0,
                                          float(tol), ctypes.byref(bad))
    if st:
        from .errors import raise_for
        raise_for(st, f"b = 0 parameters (row {bad.value})")
    p_dev = torch.from_numpy(p_host).to(v.device)
    out = check_out(out, v)
    with torch.cuda.device(v.device):
        _native.call("xft_lct_b_zero", v.data_ptr(), out.data_ptr(), B, n, _dtype_code(v), p_dev.data_ptr(),
                     0 if p_host.shape[0] == 1 else 4, _stream_ptr(v.device))
    return out
