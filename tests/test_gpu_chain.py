"""GPU parity for the composed-transform launch and the batched b = 0 branch.

* ``xft_lct_chain``: L_k ... L_1 in one launch == k sequential oracle
  ``fast_lct_rows`` calls (xft/lct.py:168-208 applied stage by stage), and the
  reference CLI's scale-adjusted inverse round trip (xft/cli.py:236-253,
  pkg/tests/test_cli.py:174-183) recovers the input.
* ``xft_lct_b_zero``: the reference's TestBZeroBranch cases
  (pkg/tests/test_lct.py:315-341) through the drop-in ``lct_b_zero`` and a
  batched per-row-parameter case against the closed form of xft/lct.py:262.

Tolerances as in test_gpu_lct.py: rel L2 <= 1e-12 (c128), <= 2e-5 (c64).
"""
import math

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import max_row_rel_l2

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


def _signal(rng, rows, n):
    x = O.asymptotic_nodes(n)
    f = np.exp(-0.5 * (x[None, :] - rng.uniform(-1, 1, (rows, 1))) ** 2) * np.exp(1j * rng.uniform(-2, 2, (rows, 1)) * x)
    return f + 0.01 * (rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n)))


STAGES = [
    [(math.cos(0.3), math.sin(0.3), -math.sin(0.3), math.cos(0.3))],
    [(1.0, 2.0, 0.5, 2.0), (0.0, 1.0, -1.0, 0.0)],
    [(0.5, 1.0, -0.25, 1.5), (math.cos(1.1), math.sin(1.1), -math.sin(1.1), math.cos(1.1)), (1.0, 0.7, 0.0, 1.0)],
    [(0.0, 1.0, -1.0, 0.0)] * 4,
]


@pytest.mark.parametrize("n", [32, 256, 1024, 4096, 8192])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("si", range(len(STAGES)))
def test_chain_matches_sequential_oracle(torch, X, n, dtype, si):
    if dtype == "c128" and n > 8192:
        pytest.skip()
    rng = np.random.default_rng(100 + n + si)
    rows = 5
    f = _signal(rng, rows, n)
    if dtype == "c64":
        f = f.astype(np.complex64)
    ref = f.astype(np.complex128)
    for p in STAGES[si]:
        ref = O.fast_lct_rows(p, ref)[1]
    scale, rev = 1.7, (si % 2 == 1)
    ref = scale * (ref[:, ::-1] if rev else ref)
    out = X.ops.lct_chain_rows(torch.from_numpy(f).cuda(), STAGES[si], scale=scale, reverse=rev)
    err = max_row_rel_l2(out.cpu().numpy().astype(np.complex128), ref)
    assert err <= (TOL128 if dtype == "c128" else TOL64), err


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_chain_16384_c64_and_rejections(torch, X, dtype):
    n = 16384 if dtype == "c64" else 8192
    rng = np.random.default_rng(7)
    f = _signal(rng, 2, n).astype(np.complex64 if dtype == "c64" else np.complex128)
    stages = [(1.0, 2.0, 0.5, 2.0), (0.0, 1.0, -1.0, 0.0)]
    ref = f.astype(np.complex128)
    for p in stages:
        ref = O.fast_lct_rows(p, ref)[1]
    out = X.ops.lct_chain_rows(torch.from_numpy(f).cuda(), stages)
    err = max_row_rel_l2(out.cpu().numpy().astype(np.complex128), ref)
    assert err <= (TOL128 if dtype == "c128" else TOL64), err
    v = torch.from_numpy(f).cuda()
    with pytest.raises(X.errors.ParameterError):
        X.ops.lct_chain_rows(v, [(1.0, 2.0, 0.5, 2.5)])          # det != 1
    with pytest.raises(X.errors.DegenerateParameterError):
        X.ops.lct_chain_rows(v, [(1.0, 0.0, 0.5, 1.0)])          # b == 0
    with pytest.raises(X.errors.ParameterError):
        X.ops.lct_chain_rows(v, [(0.0, 1.0, -1.0, 0.0)] * 5)    # > 4 stages


@pytest.mark.parametrize("n", [256, 4096])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_inverse_roundtrip_recovers_input(torch, X, n, dtype):
    """pkg/tests/test_cli.py:174-178: gaussian:1,0.3,0.1 at (1,2,0.5,2), n=256, max abs <= 1e-10."""
    x = O.asymptotic_nodes(n)
    g = np.exp(-1.0 * (x - 0.3) ** 2 + 0.1j * x)
    rows = np.stack([g, np.roll(g, 3)])
    f = rows.astype(np.complex64 if dtype == "c64" else np.complex128)
    abcd = (1.0, 2.0, 0.5, 2.0)
    out = X.ops.inverse_roundtrip_rows(torch.from_numpy(f).cuda(), abcd).cpu().numpy()
    # against the oracle's two-stage restatement of _inverse_roundtrip
    sigma = 4.0 * abcd[1] / math.pi
    second = (abcd[3] * sigma, -abcd[1] / sigma, -abcd[2] * sigma, abcd[0] / sigma)
    ref = math.sqrt(sigma) * O.fast_lct_rows(second, O.fast_lct_rows(abcd, f.astype(np.complex128))[1])[1][:, ::-1]
    err = max_row_rel_l2(out.astype(np.complex128), ref)
    assert err <= (TOL128 if dtype == "c128" else TOL64), err
    if dtype == "c128" and n == 256:
        assert np.max(np.abs(out[0] - g)) <= 1e-10
    with pytest.raises(X.errors.ParameterError):
        X.ops.inverse_roundtrip_rows(torch.from_numpy(f).cuda(), (1.0, -2.0, 0.5, -2.25 + 3.25))


# ---------------------------------------------------------------- b = 0 branch
def test_b_zero_reference_cases(torch, X):
    """pkg/tests/test_lct.py:315-341 through the drop-in lct_b_zero."""
    LctParams = X.LctParams
    res = X.lct_b_zero(LctParams(1.0, 0.0, 0.0, 1.0), lambda x: np.exp(-(x ** 2)) + 0j, 16)
    assert np.max(np.abs(res.values - np.exp(-(res.output_nodes ** 2)))) == 0.0
    res = X.lct_b_zero(LctParams(0.5, 0.0, 0.0, 2.0), lambda x: np.exp(-(x ** 2)), 32)
    expected = math.sqrt(2) * np.exp(-4.0 * res.output_nodes ** 2)
    assert np.max(np.abs(res.values - expected)) <= 1e-14
    res = X.lct_b_zero(LctParams(1.0, 0.0, 3.0, 1.0), lambda x: np.ones_like(x, dtype=complex), 32)
    expected = np.exp(1.5j * res.output_nodes ** 2)
    assert np.max(np.abs(res.values - expected)) <= 1e-14
    assert np.max(np.abs(np.abs(res.values) - 1.0)) <= 1e-14
    with pytest.raises(X.errors.UnsupportedBranchError):
        X.lct_b_zero(LctParams(-1.0, 0.0, 0.0, -1.0), lambda x: x, 8)
    with pytest.raises(X.errors.ParameterError):
        X.lct_b_zero(LctParams.fourier(), lambda x: x, 8)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_b_zero_batched_per_row(torch, X, dtype):
    rng = np.random.default_rng(5)
    rows, n = 37, 1000
    d = rng.uniform(0.3, 3.0, rows)
    c = rng.uniform(-2, 2, rows)
    abcd = np.stack([1.0 / d, np.zeros(rows), c, d], axis=1)
    samples = rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))
    y = O.asymptotic_nodes(n)
    ref = np.sqrt(d)[:, None] * np.exp(0.5j * c[:, None] * d[:, None] * np.square(y)[None, :]) * samples
    s = samples.astype(np.complex64 if dtype == "c64" else np.complex128)
    if dtype == "c64":
        ref = np.sqrt(d)[:, None] * np.exp(0.5j * c[:, None] * d[:, None] * np.square(y)[None, :]) * s.astype(complex)
    out = X.ops.lct_b_zero_rows(torch.from_numpy(s).cuda(), abcd).cpu().numpy().astype(np.complex128)
    err = max_row_rel_l2(out, ref)
    assert err <= (1e-15 if dtype == "c128" else 1e-6), err
    bad = abcd.copy()
    bad[4, 3] = -bad[4, 3]
    bad[4, 0] = 1.0 / bad[4, 3]
    with pytest.raises(X.errors.UnsupportedBranchError):
        X.ops.lct_b_zero_rows(torch.from_numpy(s).cuda(), bad)


@pytest.mark.parametrize("n,dtype", [(1000, "c128"), (16, "c64"), (65536, "c128")])
def test_chain_sizes_beyond_one_launch(torch, X, n, dtype):
    """Rows the one-launch chain kernel does not hold (non-powers of two, short, long): staged through the
    row kernels, same semantics (scale, reverse) as the fused chain."""
    rng = np.random.default_rng(n)
    f = _signal(rng, 2, n).astype(np.complex64 if dtype == "c64" else np.complex128)
    got = X.ops.inverse_roundtrip_rows(torch.from_numpy(f).cuda(), (2.0, 1.0, 1.0, 1.0)).cpu().numpy()
    a, b, c, d = 2.0, 1.0, 1.0, 1.0
    sigma = 4.0 * b / np.pi
    ref = O.fast_lct_rows((a, b, c, d), f.astype(np.complex128))[1]
    ref = O.fast_lct_rows((d * sigma, -b / sigma, -c * sigma, a / sigma), ref)[1][:, ::-1] * np.sqrt(sigma)
    err = max_row_rel_l2(got.astype(np.complex128), ref)
    assert err <= (TOL128 if dtype == "c128" else TOL64), err
