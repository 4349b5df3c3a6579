"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference/pkg/src/xft,
which does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz: inputs plus the reference's own outputs for the
hot-path functions (fast_lct / fast_frft / xft_fourier / apply_dft /
apply_scaled_fourier / frft_matrix_asymptotic / asymptotic_zeros).  The
oracle (oracle/xft_oracle.py) is pinned against these, and the GPU parity
tests compare against them directly.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import xft  # noqa: E402  (the reference)
from paper_0912_1379_b200 import workloads  # noqa: E402  (input generators only)


def rand_c(rng, shape):
    return rng.normal(size=shape) + 1j * rng.normal(size=shape)


def random_unimodular(rng, b_low=0.1, b_high=100.0):
    # same recipe as the reference's test helper (pkg/tests/test_lct.py:31-36)
    b = rng.uniform(b_low, b_high) * rng.choice([-1.0, 1.0])
    a = rng.uniform(-2.0, 2.0)
    d = rng.uniform(-2.0, 2.0)
    c = (a * d - 1.0) / b
    return (a, b, c, d)


def lct_ref(abcd, f):
    n = f.shape[0]
    res = xft.fast_lct(xft.LctParams(*abcd), xft.Signal(xft.asymptotic_zeros(n), f))
    return res.output_nodes, res.values


def main():
    out = {}
    # ---- grids -----------------------------------------------------------
    for n in (1, 2, 3, 4, 8, 1000, 1024, 4096, 16384):
        out[f"grid_n{n}"] = xft.asymptotic_zeros(n).nodes
    # ---- DFT engine ------------------------------------------------------
    dft_ns = list(range(1, 33)) + [37, 64, 100, 128, 384, 512, 600, 1000, 1024,
                                   2048, 4096, 8192, 16384, 32768]
    for n in dft_ns:
        rng = np.random.default_rng(1000 + n)
        v = rand_c(rng, n)
        out[f"dft_in_n{n}"] = v
        for sign in (1, -1):
            out[f"dft_out_n{n}_s{sign}"] = xft.apply_dft(xft.plan_dft(n, sign), v)
    for n in (2, 4, 8, 7, 64, 1000, 4096):
        rng = np.random.default_rng(2000 + n)
        v = rand_c(rng, n)
        out[f"sf_in_n{n}"] = v
        out[f"sf_out_n{n}"] = xft.apply_scaled_fourier(v)
    # ---- fast LCT: random unimodular parameters ----------------------------
    lct_ns = [1, 2, 3, 4, 5, 6, 7, 8, 16, 32, 64, 100, 128, 256, 512, 1000, 1024,
              2048, 4096, 8192, 16384]
    for n in lct_ns:
        rng = np.random.default_rng(3000 + n)
        f = rand_c(rng, n)
        P = np.array([random_unimodular(rng) for _ in range(3)]
                     + [(0.0, 1.0, -1.0, 0.0), (1.0, 2.0, 0.5, 2.0)])
        Y = []
        V = []
        for p in P:
            y, v = lct_ref(tuple(p), f)
            Y.append(y)
            V.append(v)
        out[f"lct_in_n{n}"] = f
        out[f"lct_abcd_n{n}"] = P
        out[f"lct_y_n{n}"] = np.array(Y)
        out[f"lct_out_n{n}"] = np.array(V)
    # ---- config 1 (the PR1 oracle check) -----------------------------------
    c1 = workloads.config1()
    y, v = lct_ref(tuple(c1.abcd), c1.values[0])
    out["cfg1_in"] = c1.values[0]
    out["cfg1_abcd"] = c1.abcd
    out["cfg1_y"] = y
    out["cfg1_out"] = v
    out["cfg1_dense_out"] = xft.dense_lct_matrix(1024, xft.LctParams(*c1.abcd)).apply(c1.values[0])
    # ---- config 2: first rows of the seeded batch, c128 and c64-upcast -----
    c2 = workloads.config2(row_limit=6, dtype=np.complex128)
    out["cfg2_alpha"] = c2.extra["alpha"]
    out["cfg2_in"] = c2.values
    out["cfg2_abcd"] = c2.abcd
    out["cfg2_out"] = np.array([
        xft.fast_frft(a, xft.Signal(xft.asymptotic_zeros(4096), f)).values
        for a, f in zip(c2.extra["alpha"], c2.values)])
    in64 = c2.values.astype(np.complex64).astype(np.complex128)
    out["cfg2_out_c64in"] = np.array([
        xft.fast_frft(a, xft.Signal(xft.asymptotic_zeros(4096), f)).values
        for a, f in zip(c2.extra["alpha"], in64)])
    # ---- config 4: first rows, Fourier preset via fast_lct -----------------
    c4 = workloads.config4(row_limit=4)
    f4 = c4.values.astype(np.complex128)
    out["cfg4_in"] = c4.values
    out["cfg4_out"] = np.array([lct_ref((0.0, 1.0, -1.0, 0.0), f)[1] for f in f4])
    out["cfg4_coeffs"] = c4.extra["coeffs"]
    # ---- xft_fourier / fast_frft --------------------------------------------
    for n in (8, 96, 256):
        rng = np.random.default_rng(4000 + n)
        f = rand_c(rng, n)
        g = xft.Signal(xft.asymptotic_zeros(n), f)
        out[f"fourier_in_n{n}"] = f
        out[f"fourier_out_n{n}"] = xft.xft_fourier(g).values
        out[f"frft_out_n{n}"] = np.array([xft.fast_frft(t, g).values
                                          for t in (0.3, math.pi / 2, -0.7, 3.0)])
    # ---- Mehler complex-z fractional transform (dense reference) ------------
    for n in (2, 8, 64, 256, 1024, 4096):
        rng = np.random.default_rng(5000 + n)
        f = rand_c(rng, n)
        zs = np.array([0.0, 0.5, -0.3 + 0.4j, 0.9j, 0.97 * np.exp(2.5j), 0.99, -0.99,
                       0.6 * np.exp(-1.2j)])
        out[f"mehler_in_n{n}"] = f
        out[f"mehler_z_n{n}"] = zs
        out[f"mehler_out_n{n}"] = np.array([
            xft.frft_matrix_asymptotic(n, xft.FrftOrder(z)).apply(f) for z in zs])
    # config 3 semantics at the dense cap (n = 4096): first rows
    c3 = workloads.config3(rows=1024, n=4096, row_limit=3)
    out["cfg3s_in"] = c3.values
    out["cfg3s_z"] = c3.extra["z"]
    out["cfg3s_out"] = np.array([
        xft.frft_matrix_asymptotic(4096, xft.FrftOrder(z)).apply(f)
        for z, f in zip(c3.extra["z"], c3.values)])
    # ---- 2-D separable composition (small) ---------------------------------
    n2 = 64
    field = workloads.config5_field(n=n2).astype(np.complex128)
    abcd5 = workloads.CONFIG5_ABCD
    rows = np.array([lct_ref(abcd5, r)[1] for r in field])
    cols = np.array([lct_ref(abcd5, c)[1] for c in rows.T]).T
    out["lct2d_in"] = field
    out["lct2d_out"] = cols

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
