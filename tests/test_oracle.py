"""The CPU oracle is pinned against golden vectors produced by the reference itself."""
import math

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import max_row_rel_l2, rel_l2


def test_grid_bit_exact(golden):
    for n in (1, 2, 3, 4, 8, 1000, 1024, 4096, 16384):
        assert np.array_equal(O.asymptotic_nodes(n), golden[f"grid_n{n}"])


def test_dft_bit_exact(golden):
    ns = sorted(int(k.split("_n")[1]) for k in golden if k.startswith("dft_in_n"))
    assert len(ns) > 40
    for n in ns:
        v = golden[f"dft_in_n{n}"]
        for sign in (1, -1):
            assert np.array_equal(O.dft_rows(v, sign), golden[f"dft_out_n{n}_s{sign}"]), (n, sign)


def test_dft_vs_naive(golden):
    for n in (1, 2, 3, 7, 37, 64, 100, 1000):
        v = golden[f"dft_in_n{n}"]
        for sign in (1, -1):
            assert rel_l2(O.dft_rows(v, sign), O.naive_dft(v, sign)) < 1e-11


def test_known_answers():
    # pkg/tests/test_fftcore.py:45-52
    assert np.allclose(O.dft_rows([1.0, 1.0], 1), [2.0, 0.0], atol=1e-15)
    assert np.allclose(O.dft_rows([0, 1, 0, 0], 1), [1, 1j, -1, -1j], atol=1e-15)


def test_scaled_fourier_bit_exact(golden):
    for n in (2, 4, 8, 7, 64, 1000, 4096):
        assert np.array_equal(O.scaled_fourier_rows(golden[f"sf_in_n{n}"]), golden[f"sf_out_n{n}"])


def test_fast_lct_bit_exact(golden):
    ns = sorted(int(k.split("_n")[1]) for k in golden if k.startswith("lct_in_n"))
    for n in ns:
        f = golden[f"lct_in_n{n}"]
        P = golden[f"lct_abcd_n{n}"]
        y, v = O.fast_lct_rows(P, np.broadcast_to(f, (P.shape[0], n)))
        assert np.array_equal(y, golden[f"lct_y_n{n}"]), n
        assert np.array_equal(v, golden[f"lct_out_n{n}"]), n


def test_config1_bit_exact_and_dense(golden):
    y, v = O.fast_lct_rows(golden["cfg1_abcd"], golden["cfg1_in"])
    assert np.array_equal(v, golden["cfg1_out"])
    assert np.array_equal(y, golden["cfg1_y"])
    assert rel_l2(v, golden["cfg1_dense_out"]) < 1e-12


def test_config2_rows_bit_exact(golden):
    _, v = O.fast_lct_rows(golden["cfg2_abcd"], golden["cfg2_in"])
    assert np.array_equal(v, golden["cfg2_out"])
    f64 = golden["cfg2_in"].astype(np.complex64).astype(np.complex128)
    _, v = O.fast_lct_rows(golden["cfg2_abcd"], f64)
    assert np.array_equal(v, golden["cfg2_out_c64in"])


def test_config4_rows_bit_exact(golden):
    _, v = O.fast_lct_rows((0.0, 1.0, -1.0, 0.0), golden["cfg4_in"].astype(np.complex128))
    assert np.array_equal(v, golden["cfg4_out"])


def test_fourier_and_frft(golden):
    for n in (8, 96, 256):
        f = golden[f"fourier_in_n{n}"]
        _, v = O.xft_fourier_rows(f)
        assert np.array_equal(v, golden[f"fourier_out_n{n}"])
        P = np.array([O.frft_params(t) for t in (0.3, math.pi / 2, -0.7, 3.0)])
        _, v = O.fast_lct_rows(P, np.broadcast_to(f, (4, n)))
        assert np.array_equal(v, golden[f"frft_out_n{n}"])


def test_mehler_dense(golden):
    for n in (2, 8, 64, 256, 1024):
        f = golden[f"mehler_in_n{n}"]
        for z, ref in zip(golden[f"mehler_z_n{n}"], golden[f"mehler_out_n{n}"]):
            assert rel_l2(O.mehler_apply(z, f), ref) < 1e-13, (n, z)


def test_lct2d(golden):
    got = O.lct2d((1.0, 0.25, 0.0, 1.0), (1.0, 0.25, 0.0, 1.0), golden["lct2d_in"])
    assert np.array_equal(got, golden["lct2d_out"])


def test_norm_identity():
    # ||G||^2 = pi / (4|b|) ||f||^2 for every row (SURVEY 8(a) invariant)
    rng = np.random.default_rng(5)
    f = rng.normal(size=(3, 256)) + 1j * rng.normal(size=(3, 256))
    P = np.array([(1.0, 2.0, 0.5, 2.0), O.frft_params(0.01), (0.0, 1.0, -1.0, 0.0)])
    _, v = O.fast_lct_rows(P, f)
    lhs = np.sum(np.abs(v) ** 2, axis=1)
    rhs = math.pi / (4 * np.abs(P[:, 1])) * np.sum(np.abs(f) ** 2, axis=1)
    assert np.allclose(lhs, rhs, rtol=1e-12)


def test_config5_shards_are_rows_of_the_full_draw():
    from paper_0912_1379_b200 import workloads

    full = workloads.config5_field(n=128)
    part = workloads.config5_field(n=128, rows=32, row_start=64)
    assert np.array_equal(full[64:96], part)


def test_hermite_table_matches_reference_rows():
    """hermite_function_table (the config-3/4 input generator) == the reference's hermite_function_row,
    bit for bit (fixture written by tests/golden/make_hermite_golden.py running xft/hermite.py:92-112)."""
    import os

    from paper_0912_1379_b200.hermite import hermite_function_row, hermite_function_table

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "hermite_rows.npz")
    with np.load(path) as z:
        for name in ("n1024_m21", "n16384_m31", "extra_m40"):
            xs, psi = z[f"{name}_x"], z[f"{name}_psi"]
            assert np.array_equal(hermite_function_table(psi.shape[0], xs), psi), name
            assert np.array_equal(hermite_function_row(psi.shape[0], xs[3]), psi[:, 3])


def test_dense_lct_rows_matches_reference_matrix():
    """dense_lct_rows (the full-size 2-D parity checker) == rows of the reference's dense_lct_matrix,
    bit for bit (tests/golden/cli_golden.json: xft/dense.py dense_lct_matrix at n = 48)."""
    import json
    import os

    from oracle import xft_oracle as O

    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli_golden.json")))
    d = gold["oracles"]["dense_L"]
    n = d["n"]
    L = (np.array(d["re"]) + 1j * np.array(d["im"])).reshape(n, n)
    abcd = gold["oracles"]["closed_form"]["abcd"]  # the same parameters (make_cli_golden.py)
    rows = [0, 5, 17, n - 1]
    assert np.array_equal(O.dense_lct_rows(abcd, n, rows), L[rows])
