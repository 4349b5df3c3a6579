"""GPU parity for the chirp-z kernels: non-power-of-two lengths and the Mehler transform."""
import math

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import max_row_rel_l2, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    if not _t.cuda.is_available():
        pytest.skip("no CUDA device")
    return _t


@pytest.fixture(scope="module")
def X():
    import paper_0912_1379_b200 as X

    return X


def dev(torch, a, dtype=None):
    a = np.asarray(a)
    if dtype is not None:
        a = a.astype(dtype)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


NONPOW2 = [3, 5, 6, 7, 9, 10, 11, 12, 13, 15, 17, 20, 24, 31, 37, 100, 384, 600, 1000]


@pytest.mark.parametrize("n", NONPOW2)
def test_chirpz_dft_golden(torch, X, golden, n):
    v = golden[f"dft_in_n{n}"]
    for sign in (1, -1):
        plan = X.plan_dft(n, sign)
        assert plan.route == "chirp-z"
        got = X.apply_dft(plan, v)
        assert rel_l2(got, golden[f"dft_out_n{n}_s{sign}"]) <= 1e-12, (n, sign)
        got64 = X.ops.dft_rows(dev(torch, v[None], np.complex64), sign).cpu().numpy()[0]
        ref64 = O.dft_rows(v.astype(np.complex64).astype(complex), sign)
        assert rel_l2(got64, ref64) <= 2e-5, (n, sign)


def test_chirpz_batched_and_naive(torch, X):
    rng = np.random.default_rng(7)
    for n in (3, 96, 1000, 4095):
        v = rng.normal(size=(5, n)) + 1j * rng.normal(size=(5, n))
        got = X.ops.dft_rows(dev(torch, v), -1).cpu().numpy()
        ref = O.dft_rows(v, -1) if n > 1000 else O.naive_dft(v, -1)
        assert max_row_rel_l2(got, ref) <= 1e-11, n


@pytest.mark.parametrize("n", [7, 1000])
def test_chirpz_scaled_fourier_golden(torch, X, golden, n):
    got = X.apply_scaled_fourier(golden[f"sf_in_n{n}"])
    assert rel_l2(got, golden[f"sf_out_n{n}"]) <= 1e-12


@pytest.mark.parametrize("n", [3, 5, 6, 7, 100, 1000])
def test_chirpz_lct_golden(torch, X, golden, n):
    f = golden[f"lct_in_n{n}"]
    P = golden[f"lct_abcd_n{n}"]
    got = X.ops.lct_rows(dev(torch, np.broadcast_to(f, (P.shape[0], n))), P).cpu().numpy()
    assert max_row_rel_l2(got, golden[f"lct_out_n{n}"]) <= 1e-12
    got64 = X.ops.lct_rows(dev(torch, np.broadcast_to(f, (P.shape[0], n)), np.complex64), P).cpu().numpy()
    _, ref64 = O.fast_lct_rows(P, np.broadcast_to(f, (P.shape[0], n)).astype(np.complex64).astype(complex))
    assert max_row_rel_l2(got64, ref64) <= 2e-5


def test_chirpz_fourier_frft_n96(torch, X, golden):
    g = X.Signal(X.asymptotic_zeros(96), golden["fourier_in_n96"])
    assert rel_l2(X.xft_fourier(g).values, golden["fourier_out_n96"]) <= 1e-12
    for t, ref in zip((0.3, math.pi / 2, -0.7, 3.0), golden["frft_out_n96"]):
        assert rel_l2(X.fast_frft(t, g).values, ref) <= 1e-12


def test_norm_scaling_nonpow2(torch, X):
    # pkg/tests/test_lct.py:146-159 analogue: ||G||^2 = pi/(4|b|) ||f||^2
    rng = np.random.default_rng(7)
    for n in (7, 1000):
        f = rng.normal(size=n) + 1j * rng.normal(size=n)
        res = X.fast_lct(X.LctParams(1.0, 2.0, 0.5, 2.0), X.Signal(X.asymptotic_zeros(n), f))
        lhs = np.sum(np.abs(res.values) ** 2)
        rhs = math.pi / 8 * np.sum(np.abs(f) ** 2)
        assert abs(lhs - rhs) <= 1e-10 * rhs


# --------------------------------------------------------------------------
# Mehler (complex z) -- frft_matrix_asymptotic semantics
# --------------------------------------------------------------------------
def _mehler_tol(z):
    # the reference's own expo loses ~|x|^2 / |1-z^2| ulps near z = +-1
    return 2e-12 if abs(1 - z * z) < 0.05 else 1e-12


@pytest.mark.parametrize("n", [2, 8, 64, 256, 1024, 4096])
def test_mehler_golden(torch, X, golden, n):
    f = golden[f"mehler_in_n{n}"]
    zs = golden[f"mehler_z_n{n}"]
    got = X.mehler_rows(dev(torch, np.broadcast_to(f, (zs.shape[0], n))), zs).cpu().numpy()
    for g, ref, z in zip(got, golden[f"mehler_out_n{n}"], zs):
        assert rel_l2(g, ref) <= _mehler_tol(z), (n, z)
    # the drop-in object: frft_matrix_asymptotic(n, FrftOrder(z)).apply(v)
    z = zs[2]
    got1 = X.frft_matrix_asymptotic(n, X.FrftOrder(z)).apply(f)
    assert rel_l2(got1, golden[f"mehler_out_n{n}"][2]) <= 1e-12


def test_mehler_config3_rows_at_dense_cap(torch, X, golden):
    got = X.mehler_rows(dev(torch, golden["cfg3s_in"]), golden["cfg3s_z"]).cpu().numpy()
    for g, ref, z in zip(got, golden["cfg3s_out"], golden["cfg3s_z"]):
        assert rel_l2(g, ref) <= _mehler_tol(z)


def test_mehler_errors(torch, X):
    v = dev(torch, np.ones((1, 16), dtype=complex))
    with pytest.raises(X.ParameterError):
        X.FrftOrder(1.1)
    with pytest.raises(X.SingularParameterError):
        X.mehler_rows(v, 1.0)
    with pytest.raises(X.SingularParameterError):
        X.frft_matrix_asymptotic(8, X.FrftOrder(-1.0))
    with pytest.raises(X.ParameterError):
        X.mehler_rows(v.to(torch.complex64), 0.5)


def test_mehler_hermite_eigen(torch, X):
    # continuum limit: K_z psi_m ~ sqrt(2 pi) z^m psi_m (SURVEY 8(c) closed forms)
    n = 1024
    x = X.asymptotic_zeros(n).nodes
    psi = X.hermite_function_table(8, x)
    z = 0.6 * np.exp(0.7j)
    got = X.mehler_rows(dev(torch, psi.astype(complex)), z).cpu().numpy()
    for m in range(8):
        ref = math.sqrt(2 * math.pi) * z ** m * psi[m]
        assert rel_l2(got[m], ref) <= 1e-10, m


def test_mehler_config3_full(torch, X):
    """Config 3 at full size (1024 x 16384, c128): every size class, incl. the four-step rows.

    Sampled rows/outputs against the chunked dense oracle, and every row against the
    Hermite-Gaussian eigen-relation K_z psi_m ~ sqrt(2 pi) z^m psi_m (inputs are psi_m + 1e-6 noise).
    """
    from paper_0912_1379_b200 import workloads

    c3 = workloads.config3()
    z = c3.extra["z"]
    got_t = X.mehler_rows(dev(torch, c3.values), z)
    got = got_t.cpu().numpy()
    n = 16384
    # window class of each row (same rule as the library): widest windows exercise the four-step path
    gam = np.where((2 * z / (1 - z * z)).real >= 0, (1 - z) / (2 * (1 + z)), (1 + z) / (2 * (1 - z))).real
    rows = list(np.argsort(gam)[:4]) + list(np.argsort(gam)[-2:]) + [0, 1, 511]
    js = np.linspace(0, n - 1, 97).astype(int)
    js = np.unique(np.concatenate([js, n // 2 + np.arange(-40, 40, 7)]))
    for r in rows:
        ref = O.mehler_apply(z[r], c3.values[r], rows_out=js)
        assert rel_l2(got[r, js], ref) <= _mehler_tol(z[r]), (r, z[r])
    # every row: linearity M(psi + noise) = M(psi) + M(noise), and the Hermite-Gaussian
    # eigen-relation M(psi_m) ~ sqrt(2 pi) z^m psi_m (continuum limit)
    x = X.asymptotic_zeros(n).nodes
    psi = X.hermite_function_table(31, x)[c3.extra["m"]].astype(complex)
    g_psi = X.mehler_rows(dev(torch, psi), z)
    g_noise = X.mehler_rows(dev(torch, c3.values - psi), z)
    lin = ((got_t - g_psi - g_noise).abs() ** 2).sum(1).sqrt() / (got_t.abs() ** 2).sum(1).sqrt()
    assert float(lin.max()) <= 1e-12
    g_psi = g_psi.cpu().numpy()
    for r in range(z.shape[0]):
        ideal = math.sqrt(2 * math.pi) * z[r] ** c3.extra["m"][r] * psi[r]
        assert np.linalg.norm(g_psi[r] - ideal) <= 1e-6 * max(np.linalg.norm(ideal), 1e-9), r


# ---- rows beyond the in-CTA sizes: four-step convolution (non-powers of two)
# and four-step row transforms (powers of two) -------------------------------
LARGE_NONPOW2 = [(5000, np.complex128), (12000, np.complex64), (196608, np.complex128), (196608, np.complex64)]


@pytest.mark.parametrize("n,dtype", LARGE_NONPOW2)
def test_chirpz_large_lct_dft_scaled(torch, X, n, dtype):
    """Chirp-z rows whose convolution length exceeds one CTA (196608 = the reference CLI bench size,
    pkg/tests/test_cli.py:216-220): LCT, both DFT signs and the scaled Fourier against the oracle."""
    tol = 1e-12 if dtype == np.complex128 else 2e-5
    rng = np.random.default_rng(n)
    rows = 2
    f = ((rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))) / math.sqrt(2)).astype(dtype)
    al = np.array([0.7, 2.2])
    abcd = np.stack([np.cos(al), np.sin(al), -np.sin(al), np.cos(al)], 1)
    fd = dev(torch, f)
    got = X.ops.lct_rows(fd, abcd).cpu().numpy()
    _, ref = O.fast_lct_rows(abcd, f.astype(complex))
    assert max_row_rel_l2(got, ref) <= tol
    for sign in (-1, 1):
        got = X.ops.dft_rows(fd, sign).cpu().numpy()
        assert max_row_rel_l2(got, O.dft_rows(f.astype(complex), sign)) <= tol
    got = X.ops.scaled_fourier_rows(fd).cpu().numpy()
    assert max_row_rel_l2(got, O.scaled_fourier_rows(f.astype(complex))) <= tol


@pytest.mark.parametrize("n,dtype", [(65536, np.complex128), (1 << 20, np.complex128), (1 << 20, np.complex64)])
def test_large_pow2_lct(torch, X, n, dtype):
    """Power-of-two rows up to xft_max_n (2^20) through the four-step row path."""
    tol = 1e-12 if dtype == np.complex128 else 2e-5
    rng = np.random.default_rng(n + 1)
    f = ((rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))) / math.sqrt(2)).astype(dtype)
    abcd = np.array([[2.0, 1.0, 1.0, 1.0], [math.cos(1.1), math.sin(1.1), -math.sin(1.1), math.cos(1.1)]])
    got = X.ops.lct_rows(dev(torch, f), abcd).cpu().numpy()
    _, ref = O.fast_lct_rows(abcd, f.astype(complex))
    assert max_row_rel_l2(got, ref) <= tol


def test_mehler_config3_truth(torch, X):
    """Config-3 rows with unit-modulus Mehler kernels (z ~ -0.5i .. -0.65i), where the float64
    dense formula itself loses up to ~6e-13, against a long-double evaluation of the same formula
    (tests/golden/make_mehler_truth.py): the GPU result must be within 1e-12 of the truth."""
    import os

    from paper_0912_1379_b200 import workloads

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "mehler_truth_cfg3.npz"))
    c3 = workloads.config3()
    rows = [int(r) for r in g["rows"]]
    js = g["js"]
    got = X.mehler_rows(dev(torch, c3.values[rows]), c3.extra["z"][rows]).cpu().numpy()
    for i, r in enumerate(rows):
        truth = g[f"truth_{r}"]
        assert rel_l2(got[i, js], truth) <= 1e-12, (r, rel_l2(got[i, js], truth))


@pytest.mark.slow
def test_mehler_config3_every_row_against_dense_gpu_oracle(torch, X):
    """All 1024 rows x 16384 outputs of config 3 against the entry-by-entry dense Mehler product
    (``xft_dense_mehler_apply``: K_z(x_j, x_k) dx in the reference's operation order,
    xft/dense.py:122-151; no FFT, nothing shared with the windowed Bluestein kernels)."""
    from paper_0912_1379_b200 import dense, workloads

    c3 = workloads.config3()
    z = c3.extra["z"]
    v = dev(torch, c3.values)
    got = X.mehler_rows(v, z).cpu().numpy()
    worst = []
    for s in range(0, z.shape[0], 128):  # the dense product in blocks of rows (bounded memory)
        ref = dense.dense_mehler_apply(v[s:s + 128], z[s:s + 128]).cpu().numpy()
        for r in range(ref.shape[0]):
            e = rel_l2(got[s + r], ref[r])
            worst.append(e / _mehler_tol(z[s + r]))
    assert max(worst) <= 1.0, (int(np.argmax(worst)), max(worst))


def test_mehler_caller_workspace_matches_internal_scratch(torch, X):
    """xft_mehler with a caller workspace (xft_mehler_workspace_bytes; the classes run one after
    another on the caller's stream) == the default path (internal side streams and scratch)."""
    import ctypes

    from paper_0912_1379_b200 import _native, ops
    from paper_0912_1379_b200 import workloads

    c3 = workloads.config3(rows=48)
    z = c3.extra["z"]
    v = dev(torch, c3.values)
    ref = X.mehler_rows(v, z)
    n = v.shape[1]
    nbytes = int(_native.lib().xft_mehler_workspace_bytes(v.shape[0], n))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=v.device)
    out = torch.empty_like(v)
    zh = np.ascontiguousarray(np.stack([z.real, z.imag], axis=1))
    _native.call("xft_mehler", v.data_ptr(), out.data_ptr(), v.shape[0], n, zh.ctypes.data, 2, ws.data_ptr(),
                 ops._stream_ptr(v.device))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    del ctypes


def test_mehler_near_unit_z_against_long_double_truth(torch, X, golden):
    """z = +-0.99 (|1 - z^2| < 0.05, where the Mehler parity bar against the reference is 2e-12):
    against a long-double evaluation of the dense formula (tests/golden/make_mehler_truth_golden.py)
    the GPU path meets the strict 1e-12 bar -- the reference's own float64 output is ~9e-13 off."""
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mehler_truth_golden.npz")
    with np.load(path) as t:
        keys = [k for k in t.files if not k.endswith("_z")]
        assert len(keys) == 4
        for k in keys:
            n = int(k.split("_")[0][1:])
            z = t[k + "_z"][0]
            got = X.mehler_rows(dev(torch, golden[f"mehler_in_n{n}"][None, :]), [z]).cpu().numpy()[0]
            assert rel_l2(got, t[k]) <= 1e-12, (k, rel_l2(got, t[k]))
