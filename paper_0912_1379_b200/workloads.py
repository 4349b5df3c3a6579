"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference publishes no dataset or benchmark suite; its own checks use
seeded Gaussians (xft/calibration.py).  These generators pin the draw order
of SURVEY.md 8(d) so the GPU path and the CPU oracle consume identical arrays:
``rng = np.random.default_rng(seed)``; complex N(0, s2) means
``sqrt(s2/2) * (rng.standard_normal(shape) + 1j*rng.standard_normal(shape))``
(real block first, the reference's own pattern, pkg/tests/test_lct.py:40-42).

Everything here is host-side input construction, outside any timed region.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .hermite import asymptotic_zeros, hermite_function_table


def complex_normal(rng, var: float, shape) -> np.ndarray:
    s = math.sqrt(var / 2.0)
    return s * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def frft_abcd(angle: float):
    """LctParams.frft quadruple with the reference's 1e-15 snapping (xft/lct.py:97-109)."""
    ca, sa = math.cos(angle), math.sin(angle)
    if abs(ca) < 1e-15:
        ca = 0.0
    if abs(sa) < 1e-15:
        sa = 0.0
    return (ca, sa, -sa, ca)


@dataclass
class Batch1D:
    name: str
    values: np.ndarray          # (B, n) complex64 or complex128
    abcd: np.ndarray            # (B, 4) or (4,) float64
    extra: dict


def config1() -> Batch1D:
    """Single 1-D LCT, n=1024, c128, (a,b,c,d)=(2,1,1,1); f = e^{-x^2/2}(1+0.3x) + CN(0,1e-3), seed 0."""
    n = 1024
    x = asymptotic_zeros(n).nodes
    rng = np.random.default_rng(0)
    f = np.exp(-x * x / 2) * (1 + 0.3 * x) + complex_normal(rng, 1e-3, n)
    return Batch1D("cfg1", f[None, :].astype(np.complex128),
                   np.array([2.0, 1.0, 1.0, 1.0]), {})


def config2(rows: int = 4096, n: int = 4096, dtype=np.complex64, row_limit=None) -> Batch1D:
    """Batched FrFT: alpha ~ U(0, pi) per row then X ~ CN(0,1) [rows, n], seed 1.

    ``row_limit`` keeps only the first rows of the same draw (the draw
    itself always has the full shape, so the kept rows are identical).
    """
    rng = np.random.default_rng(1)
    alpha = rng.uniform(0.0, math.pi, rows)
    X = complex_normal(rng, 1.0, (rows, n))
    if row_limit is not None:
        alpha, X = alpha[:row_limit], X[:row_limit]
    abcd = np.array([frft_abcd(a) for a in alpha])
    return Batch1D("cfg2", X.astype(dtype), abcd, {"alpha": alpha})


def config3(rows: int = 1024, n: int = 16384, row_limit=None) -> Batch1D:
    """Complex-z (Mehler) FrFT: r~U(.5,.99), alpha~U(0,2pi), m~U{0..30}, noise CN(0,1e-6); seed 2."""
    rng = np.random.default_rng(2)
    r = rng.uniform(0.5, 0.99, rows)
    alpha = rng.uniform(0.0, 2 * math.pi, rows)
    m = rng.integers(0, 31, rows)
    noise = complex_normal(rng, 1e-6, (rows, n))
    if row_limit is not None:
        r, alpha, m, noise = r[:row_limit], alpha[:row_limit], m[:row_limit], noise[:row_limit]
    x = asymptotic_zeros(n).nodes
    psi = hermite_function_table(31, x)
    f = psi[m] + noise
    z = r * np.exp(1j * alpha)
    return Batch1D("cfg3", f.astype(np.complex128), np.zeros(4), {"z": z, "m": m})


def config4(rows: int = 65536, n: int = 1024, row_limit=None) -> Batch1D:
    """Fourier via XFT (0,1,-1,0): X = C @ Psi[0:21], C ~ CN(0,1) [rows, 21], seed 3; c64."""
    rng = np.random.default_rng(3)
    C = complex_normal(rng, 1.0, (rows, 21))
    if row_limit is not None:
        C = C[:row_limit]
    x = asymptotic_zeros(n).nodes
    psi = hermite_function_table(21, x)
    X = C @ psi
    return Batch1D("cfg4", X.astype(np.complex64), np.array([0.0, 1.0, -1.0, 0.0]),
                   {"coeffs": C})


def config4_closed_form(coeffs: np.ndarray, n: int = 1024) -> np.ndarray:
    """Continuous Fourier-preset transform of sum_m C_m psi_m: sum C_m e^{-i pi/4} (-i)^m psi_m(y_j).

    Output nodes y_j = (4/pi) x_j (b = 1).  Used for the quadrature-error report.
    """
    x = asymptotic_zeros(n).nodes
    y = (4.0 / math.pi) * x
    psi_y = hermite_function_table(coeffs.shape[1], y)
    phase = np.exp(-1j * math.pi / 4) * (-1j) ** np.arange(coeffs.shape[1])
    return (coeffs * phase) @ psi_y


def config5_field(n: int = 16384, rows=None, out=None, row_start: int = 0) -> np.ndarray:
    """Random-phase disk aperture, radius 0.3 * (x[-1]-x[0]), phase ~ U(0, 2pi) [n, n], seed 4; c64.

    Drawn row block by row block (the uniform stream is consumed in the same
    row-major order as one (n, n) draw).  ``row_start``/``rows`` select a row
    shard: the generator is advanced past the earlier rows (one 64-bit draw
    per uniform double), so every shard is bit-identical to the same rows of
    the full draw.
    """
    x = asymptotic_zeros(n).nodes
    extent = x[-1] - x[0]
    R = 0.3 * extent
    nrows = (n - row_start) if rows is None else rows
    field = out if out is not None else np.empty((nrows, n), dtype=np.complex64)
    rng = np.random.default_rng(4)
    if row_start:
        rng.bit_generator.advance(row_start * n)
    blk = 256
    x2 = x * x
    for s in range(0, nrows, blk):
        e = min(s + blk, nrows)
        phase = rng.uniform(0.0, 2 * math.pi, (e - s, n))
        gs, ge = row_start + s, row_start + e
        inside = (x2[gs:ge, None] + x2[None, :]) <= R * R
        field[s:e] = (inside * np.exp(1j * phase)).astype(np.complex64)
    return field


CONFIG5_ABCD = (1.0, 0.25, 0.0, 1.0)
