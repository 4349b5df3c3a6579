"""CPU oracle for the XFT fast-LCT hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference algorithm
(``/root/reference/pkg/src/xft``, cited below as ``xft/<file>:<line>``).  It is
the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package (``paper_0912_1379_b200``) never imports this file and has
no CPU fallback.

Parity pin: every function here is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/xft`` and writes ``tests/golden/*.npz``); the
radix-2 / chirp-z DFT, grid, chirp and LCT restatements reproduce the
reference **bit for bit** on those vectors (``tests/test_oracle.py``).

All transforms are row-batched: a ``[B, n]`` complex128 array is processed
row by row with exactly the reference's elementwise operation order, so each
row is bit-identical to a reference call on that row.
"""
from __future__ import annotations

import math

import numpy as np

DFT_SIGN = -1  # xft/kernel.py:42


# --------------------------------------------------------------------------
# grid (xft/hermite.py:74-89)
# --------------------------------------------------------------------------
def grid_spacing(n: int) -> float:
    """pi / sqrt(2n)  (xft/hermite.py:74-77)."""
    return math.pi / math.sqrt(2.0 * n)


def asymptotic_nodes(n: int) -> np.ndarray:
    """x_k = (2k - n + 1) * half, half = spacing / 2  (xft/hermite.py:80-89)."""
    half = grid_spacing(n) / 2.0
    offsets = 2 * np.arange(n) - (n - 1)
    return offsets * half


# --------------------------------------------------------------------------
# kernel factors (xft/kernel.py:45-113)
# --------------------------------------------------------------------------
def kernel_prefactor(n: int) -> complex:
    """C(n) = pi/sqrt(2n) * exp(-i pi ((n-1)^2 mod 4n) / (2n))  (xft/kernel.py:45-48)."""
    red = ((n - 1) * (n - 1)) % (4 * n)
    return np.pi / np.sqrt(2.0 * n) * np.exp(DFT_SIGN * 1j * np.pi * red / (2.0 * n))


def boundary_phase(n: int) -> np.ndarray:
    """p_k = exp(+i pi ((n-1) k mod 2n) / n)  (xft/kernel.py:51-65)."""
    k = np.arange(n, dtype=np.int64)
    red = ((n - 1) * k) % (2 * n)
    return np.exp(-DFT_SIGN * 1j * np.pi * red.astype(float) / n)


def input_chirp(a: float, b: float, x: np.ndarray) -> np.ndarray:
    """exp(i a x^2 / (2b))  (xft/kernel.py:98-102)."""
    return np.exp((0.5j * a / b) * np.square(x))


def output_chirp(d: float, b: float, y: np.ndarray) -> np.ndarray:
    """exp(i d y^2 / (2b)) / sqrt(2 pi i b)  (xft/kernel.py:105-113)."""
    return np.exp((0.5j * d / b) * np.square(y)) / np.sqrt(2j * np.pi * b)


# --------------------------------------------------------------------------
# DFT engine (xft/fftcore.py:24-137)
# --------------------------------------------------------------------------
def _bit_reverse_indices(n: int) -> np.ndarray:
    """xft/fftcore.py:24-30."""
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        rev = (rev << 1) | ((idx >> b) & 1)
    return rev


def _pow2_tables(n: int, sign: int):
    """xft/fftcore.py:33-40."""
    rev = _bit_reverse_indices(n)
    twiddles = []
    m = 1
    while m < n:
        twiddles.append(np.exp(sign * 1j * np.pi * np.arange(m) / m))
        m *= 2
    return rev, tuple(twiddles)


def _apply_pow2_rows(v: np.ndarray, rev, twiddles) -> np.ndarray:
    """Radix-2 DIT over the last axis (xft/fftcore.py:43-54), batched over rows."""
    rows = v.shape[0]
    a = v[:, rev]
    m = 1
    for w in twiddles:
        a = a.reshape(rows, -1, 2, m)
        t = a[:, :, 1, :] * w
        top = a[:, :, 0, :] + t
        a[:, :, 1, :] = a[:, :, 0, :] - t
        a[:, :, 0, :] = top
        a = a.reshape(rows, -1)
        m *= 2
    return a


def dft_rows(v: np.ndarray, sign: int) -> np.ndarray:
    """Unnormalised DFT out[j] = sum_k exp(sign 2 pi i jk/n) v[k] per row.

    Route selection as DftPlan (xft/fftcore.py:73-100): radix-2 for powers
    of two, Bluestein chirp-z into a power-of-two circular convolution
    otherwise (xft/fftcore.py:84-100, 116-119).
    """
    v = np.array(v, dtype=complex, copy=True)
    squeeze = v.ndim == 1
    if squeeze:
        v = v[None, :]
    n = v.shape[1]
    if n & (n - 1) == 0:
        out = _apply_pow2_rows(v, *_pow2_tables(n, sign))
    else:
        m = 1
        while m < 2 * n - 1:
            m *= 2
        k = np.arange(n, dtype=np.int64)
        chirp = np.exp(sign * 1j * np.pi * ((k * k) % (2 * n)) / n)
        filt = np.zeros(m, dtype=complex)
        filt[:n] = np.conj(chirp)
        filt[m - n + 1:] = np.conj(chirp[1:][::-1])
        fwd = _pow2_tables(m, -1)
        inv = _pow2_tables(m, +1)
        filter_fft = _apply_pow2_rows(filt[None, :], *fwd)[0]
        u = np.zeros((v.shape[0], m), dtype=complex)
        u[:, :n] = v * chirp
        conv = _apply_pow2_rows(_apply_pow2_rows(u, *fwd) * filter_fft, *inv)
        out = chirp * conv[:, :n] / m
    return out[0] if squeeze else out


def naive_dft(v, sign: int) -> np.ndarray:
    """O(n^2) DFT (xft/fftcore.py:122-137), used to cross-check dft_rows."""
    v = np.asarray(v, dtype=complex)
    n = v.shape[-1]
    j = np.arange(n, dtype=np.int64)
    kernel = np.exp(sign * 2j * np.pi * (np.outer(j, j) % n) / n)
    return v @ kernel.T


# --------------------------------------------------------------------------
# fast LCT (xft/lct.py:168-233)
# --------------------------------------------------------------------------
def _abcd_rows(abcd, rows: int) -> np.ndarray:
    p = np.asarray(abcd, dtype=np.float64)
    if p.ndim == 1:
        p = np.broadcast_to(p, (rows, 4))
    return p


def frft_params(angle: float):
    """LctParams.frft (xft/lct.py:97-109): snaps |cos|,|sin| < 1e-15 to 0."""
    ca, sa = math.cos(angle), math.sin(angle)
    if abs(ca) < 1e-15:
        ca = 0.0
    if abs(sa) < 1e-15:
        sa = 0.0
    return (ca, sa, -sa, ca)


def fast_lct_rows(abcd, f: np.ndarray):
    """Batched restatement of fast_lct (xft/lct.py:168-208).

    ``abcd``: (4,) or (B, 4) float64; ``f``: (B, n) or (n,) complex.
    Returns (y, values) with y of shape (B, n) (per-row output nodes
    y_j = 4 b x_j / pi, xft/lct.py:196) and values complex128.
    No validation: the checker assumes valid parameters.
    """
    f = np.asarray(f)
    squeeze = f.ndim == 1
    f2 = (f[None, :] if squeeze else f).astype(complex)
    rows, n = f2.shape
    p_rows = _abcd_rows(abcd, rows)
    x = asymptotic_nodes(n)
    p = boundary_phase(n)
    cn = kernel_prefactor(n)
    u = np.empty_like(f2)
    ys = np.empty((rows, n))
    post = np.empty_like(f2)
    for r in range(rows):
        a, b, _c, d = (float(t) for t in p_rows[r])
        y = (4.0 * b / np.pi) * x                       # xft/lct.py:196
        u[r] = p * input_chirp(a, b, x) * f2[r]          # xft/lct.py:204-205
        ys[r] = y
        post[r] = cn * p * output_chirp(d, b, y)         # xft/lct.py:207 (factor part)
    spectrum = dft_rows(u, DFT_SIGN)                     # xft/lct.py:206
    values = post * spectrum                             # xft/lct.py:207
    if squeeze:
        return ys[0], values[0]
    return ys, values


def xft_fourier_rows(f: np.ndarray):
    """sqrt(2 pi i) * fast_lct at (0,1,-1,0)  (xft/lct.py:211-223)."""
    y, v = fast_lct_rows((0.0, 1.0, -1.0, 0.0), f)
    return y, np.sqrt(2j * np.pi) * v


def scaled_fourier_rows(v: np.ndarray) -> np.ndarray:
    """apply_scaled_fourier: C(n) (p * DFT(p * v))  (xft/kernel.py:83-95)."""
    v = np.asarray(v, dtype=complex)
    n = v.shape[-1]
    p = boundary_phase(n)
    return kernel_prefactor(n) * (p * dft_rows(p * v, DFT_SIGN))


def dense_lct_rows(abcd, n: int, rows) -> np.ndarray:
    """Selected rows j of the dense LCT matrix, in the reference's operation order
    (dense_lct_matrix, xft/dense.py:162-171; scaled_fourier_matrix, xft/kernel.py:68-80):
    L[j, k] = oc_j * (C(n) * (p_j * e^{-2 pi i (jk mod n)/n} * p_k)) * ic_k.
    Any n (the reference caps the materialised matrix at 4096; one row is O(n))."""
    a, b, _c, d = (float(t) for t in abcd)
    js = np.asarray(rows, dtype=np.int64)
    x = asymptotic_nodes(n)
    y = (4.0 * b / np.pi) * x
    k = np.arange(n, dtype=np.int64)
    dft = np.exp(DFT_SIGN * 2j * np.pi * ((js[:, None] * k[None, :]) % n) / n)
    p = boundary_phase(n)
    f = kernel_prefactor(n) * (p[js][:, None] * dft * p[None, :])
    return output_chirp(d, b, y)[js][:, None] * f * input_chirp(a, b, x)[None, :]


def lct2d(abcd_row, abcd_col, field: np.ndarray) -> np.ndarray:
    """Separable 2-D LCT: fast_lct along axis 1, then along axis 0.

    There is no reference symbol; this is the composition of the 1-D
    reference transform (xft/lct.py:168-208) along both axes.
    """
    _, g = fast_lct_rows(abcd_row, field)
    _, h = fast_lct_rows(abcd_col, np.ascontiguousarray(g.T))
    return np.ascontiguousarray(h.T)


# --------------------------------------------------------------------------
# Mehler kernel / complex-z fractional transform (xft/dense.py:122-151)
# --------------------------------------------------------------------------
def mehler_kernel(z: complex, x, y):
    """K_z(x, y) (xft/dense.py:122-136), principal sqrt branch."""
    z = complex(z)
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    one = 1.0 - z * z
    expo = -((1.0 + z * z) * (x * x + y * y) - 4.0 * x * y * z) / (2.0 * one)
    return np.sqrt(2.0 / one) * np.exp(expo)


def mehler_apply(z: complex, f: np.ndarray, rows_out=None, chunk: int = 256) -> np.ndarray:
    """g = (K_z(x_j, x_k) * dx) @ f  (xft/dense.py:139-151 + 76-80).

    Chunked over output rows j so it runs beyond the reference's n <= 4096
    memory guard (xft/dense.py:44, 83-89); ``rows_out`` selects a subset of
    output indices j (default: all).
    """
    f = np.asarray(f, dtype=complex)
    n = f.shape[0]
    x = asymptotic_nodes(n)
    dx = grid_spacing(n)
    js = np.arange(n) if rows_out is None else np.asarray(rows_out)
    out = np.empty(js.shape[0], dtype=complex)
    for s in range(0, js.shape[0], chunk):
        jj = js[s:s + chunk]
        ent = mehler_kernel(z, x[jj][:, None], x[None, :]) * dx
        out[s:s + chunk] = ent @ f
    return out
