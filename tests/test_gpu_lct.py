"""GPU parity: the CUDA path against reference golden vectors and the CPU oracle.

Tolerances (north star, BASELINE.json): per-row relative L2 <= 1e-12 for
complex128, <= 2e-5 for complex64 (oracle fed the c64 data upcast to c128).
"""
import math

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import max_row_rel_l2, rel_l2

pytestmark = pytest.mark.gpu

TOL128 = 1e-12
TOL64 = 2e-5


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


def lct_gpu(torch, X, abcd, f, dtype=np.complex128, **kw):
    f = np.atleast_2d(f)
    return X.ops.lct_rows(dev(torch, f, dtype), abcd, **kw).cpu().numpy()


# --------------------------------------------------------------------------
# golden vectors from the reference
# --------------------------------------------------------------------------
LCT_NS = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384]


@pytest.mark.parametrize("n", LCT_NS)
def test_lct_golden_c128(torch, X, golden, n):
    if n > X._native.lib().xft_max_n(1):
        pytest.skip("c128 row longer than the single-CTA path")
    f = golden[f"lct_in_n{n}"]
    P = golden[f"lct_abcd_n{n}"]
    got = lct_gpu(torch, X, P, np.broadcast_to(f, (P.shape[0], n)))
    assert max_row_rel_l2(got, golden[f"lct_out_n{n}"]) <= TOL128


@pytest.mark.parametrize("n", LCT_NS)
def test_lct_golden_c64(torch, X, golden, n):
    f = golden[f"lct_in_n{n}"]
    P = golden[f"lct_abcd_n{n}"]
    f64 = np.broadcast_to(f, (P.shape[0], n)).astype(np.complex64)
    got = lct_gpu(torch, X, P, f64, dtype=np.complex64)
    _, ref = O.fast_lct_rows(P, f64.astype(np.complex128))
    assert max_row_rel_l2(got, ref) <= TOL64


POW2 = [1, 2, 4, 8, 16, 32, 64, 128, 512, 1024, 2048, 4096, 8192, 16384, 32768]


@pytest.mark.parametrize("n", POW2)
def test_dft_golden(torch, X, golden, n):
    v = golden[f"dft_in_n{n}"]
    for sign in (1, -1):
        ref = golden[f"dft_out_n{n}_s{sign}"]
        if n <= X._native.lib().xft_max_n(1):
            got = X.ops.dft_rows(dev(torch, v[None]), sign).cpu().numpy()[0]
            assert rel_l2(got, ref) <= 1e-13, (n, sign)
        got = X.ops.dft_rows(dev(torch, v[None], np.complex64), sign).cpu().numpy()[0]
        ref64 = O.dft_rows(v.astype(np.complex64).astype(complex), sign)
        assert rel_l2(got, ref64) <= 1e-5, (n, sign)


def test_dft_known_answers(torch, X):
    # pkg/tests/test_fftcore.py:45-52
    for sign in (1, -1):
        out = X.apply_dft(X.plan_dft(2, sign), [1.0, 1.0])
        assert np.allclose(out, [2.0, 0.0], atol=1e-15)
    out = X.apply_dft(X.plan_dft(4, 1), [0, 1, 0, 0])
    assert np.allclose(out, [1, 1j, -1, -1j], atol=1e-15)
    assert X.apply_dft(X.plan_dft(1, 1), [3.0 - 1j]).tolist() == [3.0 - 1j]


@pytest.mark.parametrize("n", [2, 4, 8, 64, 4096])
def test_scaled_fourier_golden(torch, X, golden, n):
    got = X.apply_scaled_fourier(golden[f"sf_in_n{n}"])
    assert rel_l2(got, golden[f"sf_out_n{n}"]) <= TOL128


# --------------------------------------------------------------------------
# BASELINE configs
# --------------------------------------------------------------------------
def test_config1(torch, X, golden):
    got = lct_gpu(torch, X, golden["cfg1_abcd"], golden["cfg1_in"])[0]
    assert rel_l2(got, golden["cfg1_out"]) <= TOL128
    assert rel_l2(got, golden["cfg1_dense_out"]) <= TOL128


def test_config2_rows_golden(torch, X, golden):
    got = lct_gpu(torch, X, golden["cfg2_abcd"], golden["cfg2_in"])
    assert max_row_rel_l2(got, golden["cfg2_out"]) <= TOL128
    got = lct_gpu(torch, X, golden["cfg2_abcd"], golden["cfg2_in"], dtype=np.complex64)
    assert max_row_rel_l2(got, golden["cfg2_out_c64in"]) <= TOL64


def test_config4_rows_golden(torch, X, golden):
    got = lct_gpu(torch, X, (0.0, 1.0, -1.0, 0.0), golden["cfg4_in"], dtype=np.complex64)
    assert max_row_rel_l2(got, golden["cfg4_out"]) <= TOL64


@pytest.mark.parametrize("dtype,tol", [(np.complex64, TOL64), (np.complex128, TOL128)])
def test_config2_full_batch(torch, X, dtype, tol):
    """Full 4096 x 4096 batch: EVERY row against the oracle (chunked) + the norm identity on all rows."""
    from paper_0912_1379_b200 import workloads

    c2 = workloads.config2(dtype=dtype)
    got_t = X.ops.lct_rows(dev(torch, c2.values), c2.abcd)
    got_all = got_t.cpu().numpy()
    worst = 0.0
    for r0 in range(0, c2.values.shape[0], 512):
        _, ref = O.fast_lct_rows(c2.abcd[r0:r0 + 512], c2.values[r0:r0 + 512].astype(np.complex128))
        worst = max(worst, max_row_rel_l2(got_all[r0:r0 + 512], ref))
    assert worst <= tol, worst
    # ||G||^2 = pi/(4|b|) ||f||^2 on every row
    f = dev(torch, c2.values).to(torch.complex128)
    lhs = (got_t.to(torch.complex128).abs() ** 2).sum(dim=1).cpu().numpy()
    rhs = (math.pi / (4 * np.abs(c2.abcd[:, 1]))) * (f.abs() ** 2).sum(dim=1).cpu().numpy()
    assert np.max(np.abs(lhs / rhs - 1)) <= (1e-12 if dtype == np.complex128 else 1e-4)


@pytest.mark.parametrize("n", [64, 1024, 4096, 8192])
def test_c128_chirp_modes(torch, X, n):
    """c128 rows whose largest chirp phase puts each side in every evaluation mode:
    smooth walk (< 2^13 rad, incl. rows just below the threshold), walk + per-element
    rounding correction (< 2^24), table (< 1e12), pre-reduced table (beyond), and
    a = 0 / d = 0 rows."""
    rows = []
    xm2 = ((n - 1) * math.pi / math.sqrt(2 * n) / 2) ** 2  # largest x^2 on the grid
    edge = [math.atan(0.5 * xm2 / p) for p in (8150.0, 8250.0)]  # max |phase| just below / above 2^13
    for al in (math.pi / 2, 1.3, 0.3, 3.02e-4, math.pi - 6.56e-4, 1e-6, 1e-10, *edge):
        rows.append((math.cos(al), math.sin(al), -math.sin(al), math.cos(al)))
    for a, b, d in ((2.0, 1.0, 2000.0), (0.5, 1.0, 1e6), (3.0, 1.0, 1e10), (1e8, 1.0, 0.0), (0.0, 1.0, 1e7),
                    (-2.5, -0.7, 33.0)):
        rows.append((a, b, (a * d - 1.0) / b, d))
    abcd = np.array(rows, dtype=np.float64)
    rng = np.random.default_rng(11)
    f = (rng.standard_normal((len(rows), n)) + 1j * rng.standard_normal((len(rows), n))) / math.sqrt(2)
    got = X.ops.lct_rows(dev(torch, f), abcd).cpu().numpy()
    _, ref = O.fast_lct_rows(abcd, f)
    err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert np.max(err) <= TOL128, err


def test_config4_full_batch_and_quadrature(torch, X):
    from paper_0912_1379_b200 import workloads

    c4 = workloads.config4()
    got_t = X.ops.lct_rows(dev(torch, c4.values), c4.abcd)
    got_all = got_t.cpu().numpy()
    worst = 0.0
    for r0 in range(0, c4.values.shape[0], 8192):  # every one of the 65536 rows against the oracle
        _, ref = O.fast_lct_rows(c4.abcd, c4.values[r0:r0 + 8192].astype(np.complex128))
        worst = max(worst, max_row_rel_l2(got_all[r0:r0 + 8192], ref))
    assert worst <= TOL64, worst
    rows = [0, 1, 777, 65535]
    got = got_all[rows]
    # the continuous transform of the Hermite-Gaussian mixture (quadrature error report)
    cf = workloads.config4_closed_form(c4.extra["coeffs"][rows])
    lo, hi = 1024 // 10, 9 * 1024 // 10
    assert np.max(np.abs(got[:, lo:hi] - cf[:, lo:hi])) <= 1e-4 * np.max(np.abs(cf))


# --------------------------------------------------------------------------
# reference API behaviour (pkg/tests/test_lct.py, test_fftcore.py analogues)
# --------------------------------------------------------------------------
def test_fourier_and_frft_golden(torch, X, golden):
    for n in (8, 96, 256):
        g = X.Signal(X.asymptotic_zeros(n), golden[f"fourier_in_n{n}"]) if n != 96 else None
        if g is None:
            continue  # n = 96 is not a power of two (chirp-z route, see test_bluestein)
        assert rel_l2(X.xft_fourier(g).values, golden[f"fourier_out_n{n}"]) <= TOL128
        for t, ref in zip((0.3, math.pi / 2, -0.7, 3.0), golden[f"frft_out_n{n}"]):
            assert rel_l2(X.fast_frft(t, g).values, ref) <= TOL128


def test_quarter_turn_bitwise_equals_fourier(torch, X):
    rng = np.random.default_rng(31)
    g = X.Signal(X.asymptotic_zeros(64), rng.normal(size=64) + 1j * rng.normal(size=64))
    a = X.fast_frft(math.pi / 2, g)
    b = X.fast_lct(X.LctParams.fourier(), g)
    assert np.array_equal(a.values, b.values)


def test_zero_in_zero_out(torch, X):
    for n in (16, 1024):
        g = X.Signal(X.asymptotic_zeros(n), np.zeros(n, dtype=complex))
        assert np.all(X.fast_lct(X.LctParams(1.0, 2.0, 0.5, 2.0), g).values == 0)
        assert np.all(X.xft_fourier(g).values == 0)


def test_deterministic_and_input_untouched(torch, X):
    rng = np.random.default_rng(4)
    v = dev(torch, rng.normal(size=(64, 4096)) + 1j * rng.normal(size=(64, 4096)), np.complex64)
    keep = v.clone()
    P = np.array([X.LctParams.frft(0.1 + 0.01 * i).as_tuple() for i in range(64)])
    a = X.ops.lct_rows(v, P)
    b = X.ops.lct_rows(v, P)
    assert torch.equal(a, b)
    assert torch.equal(v, keep)


def test_output_nodes_and_validation_order(torch, X):
    g = X.Signal(X.asymptotic_zeros(4), np.ones(4, dtype=complex))
    with pytest.raises(X.DegenerateParameterError):
        X.fast_lct(X.LctParams(1.0, 0.0, 0.0, 1.0), g)
    with pytest.raises(X.ParameterError):
        X.fast_lct(X.LctParams(1.0, 1.0, 1.0, 1.0), g)
    X.fast_lct(X.LctParams(1.0, 1.0, 1.0, 1.0), g, check_unimodular=False)
    nodes = np.linspace(-1, 1, 8)
    bad = X.HermiteGrid(n=8, nodes=nodes, spacing=nodes[1] - nodes[0])
    with pytest.raises(X.GridMismatchError):
        X.fast_lct(X.LctParams.fourier(), X.Signal(bad, np.ones(8, dtype=complex)))
    with pytest.raises(X.ShapeError):
        X.fast_lct(X.LctParams.fourier(), X.Signal(X.asymptotic_zeros(8), np.ones(8)),
                   plan=X.plan_dft(16, -1))
    with pytest.raises(X.DegenerateParameterError):
        X.fast_frft(0.0, g)
    rng = np.random.default_rng(0)
    sig = X.Signal(X.asymptotic_zeros(32), rng.normal(size=32) + 0j)
    p = X.LctParams(1.0, -2.5, (0.6 - 1) / -2.5, 0.6)
    res = X.fast_lct(p, sig)
    assert np.max(np.abs(res.output_nodes - (4 * p.b / np.pi) * sig.grid.nodes)) <= 1e-13


def test_batch_param_errors(torch, X):
    v = dev(torch, np.ones((3, 8)), np.complex128)
    P = np.array([X.LctParams.frft(0.3).as_tuple(), (1.0, 0.0, 0.0, 1.0), (1.0, 1.0, 1.0, 1.0)])
    with pytest.raises(X.DegenerateParameterError):   # b == 0 checked before unimodularity
        X.ops.lct_rows(v, P)
    P[1] = X.LctParams.frft(0.2).as_tuple()
    with pytest.raises(X.ParameterError):
        X.ops.lct_rows(v, P)


def test_host_end_to_end_matches_device(torch, X):
    from paper_0912_1379_b200 import workloads

    c2 = workloads.config2(rows=512, n=4096, dtype=np.complex64, row_limit=None)
    host_in = torch.from_numpy(c2.values).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    X.ops.lct_host(host_in.numpy(), c2.abcd, out=host_out.numpy())
    ref = X.ops.lct_rows(dev(torch, c2.values), c2.abcd).cpu()
    assert torch.equal(host_out, ref)
    with pytest.raises(X.DegenerateParameterError):
        X.ops.lct_host(c2.values[:2], (1.0, 0.0, 0.0, 1.0))


def test_empty_batch(torch, X):
    v = torch.empty((0, 64), dtype=torch.complex128, device="cuda")
    assert X.ops.lct_rows(v, (0.0, 1.0, -1.0, 0.0)).shape == (0, 64)


def test_lct2d_golden(torch, X, golden):
    from paper_0912_1379_b200 import lct2d

    f = dev(torch, golden["lct2d_in"])
    got = lct2d.lct2d(f, (1.0, 0.25, 0.0, 1.0), (1.0, 0.25, 0.0, 1.0)).cpu().numpy()
    assert rel_l2(got, golden["lct2d_out"]) <= TOL128


@pytest.mark.parametrize("n", [16, 1000, 4096, 8192, 16384, 32768])
@pytest.mark.parametrize("dt", ["c64", "c128"])
def test_nonfinite_rows_reported(torch, n, dt):
    """check_finite: the reference's Signal check (xft/lct.py:125-126) on a batch -- fused into the
    pipelined row kernel, a pre-scan on the short-row / chirp-z / four-step paths."""
    from paper_0912_1379_b200 import ops
    from paper_0912_1379_b200.errors import ParameterError

    dtype = torch.complex64 if dt == "c64" else torch.complex128
    rng = np.random.default_rng(n)
    x = torch.from_numpy(rng.normal(size=(12, n)) + 1j * rng.normal(size=(12, n))).to(dtype).cuda()
    p = (0.6, 0.8, -0.8, 0.6)
    ref = ops.lct_rows(x, p)
    assert torch.equal(ops.lct_rows(x, p, check_finite=True), ref)  # finite batch: same result
    big = x.clone()
    big[3, 7] = complex(1e300, -1e300) if dt == "c128" else complex(1e30, -1e30)  # finite: accepted
    ops.lct_rows(big, p, check_finite=True)
    for bad_val, rows in ((float("nan"), (9, 5)), (float("inf"), (11,)), (complex(0, -float("inf")), (2, 10))):
        y = x.clone()
        for r in rows:
            y[r, (r * 37) % n] = bad_val
        with pytest.raises(ParameterError, match=f"row {min(rows)}"):
            ops.lct_rows(y, p, check_finite=True)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 600, 1000, 4096])
@pytest.mark.parametrize("sign", [1, -1])
def test_naive_dft_matches_oracle(torch, X, n, sign):
    """naive_dft (xft/fftcore.py:122-137) on the GPU, entry by entry: vs the oracle's naive DFT and
    the reference's known answers (pkg/tests/test_fftcore.py:45-52)."""
    from oracle import xft_oracle as O

    rng = np.random.default_rng(n + sign)
    v = rng.normal(size=n) + 1j * rng.normal(size=n)
    got = X.naive_dft(v, sign)
    ref = O.naive_dft(v, sign)
    assert rel_l2(got, ref) <= 1e-13
    assert np.allclose(X.naive_dft(np.ones(2), -1), [2, 0], atol=1e-15)
    assert np.allclose(X.naive_dft(np.array([0, 1, 0, 0]), -1), [1, -1j, -1, 1j], atol=1e-15)


def test_naive_dft_errors(torch, X):
    with pytest.raises(X.ParameterError):
        X.naive_dft(np.ones(4), 0)
    with pytest.raises(X.InvalidSizeError):
        X.naive_dft(np.ones(0), 1)
    with pytest.raises(X.InvalidSizeError):
        X.naive_dft(np.ones(4097), 1)
