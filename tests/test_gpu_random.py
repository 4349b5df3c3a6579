"""Randomised parity sweep (seeded): row lengths across every code path (single-pass, in-CTA
pipelined, four-step, chirp-z in one CTA and four-step), random unimodular parameters of
either sign, both dtypes, against the CPU oracle."""
import math

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import max_row_rel_l2

pytestmark = pytest.mark.gpu

LENGTHS = [2, 3, 8, 16, 17, 31, 64, 100, 256, 384, 1000, 1024, 2047, 4096, 5000, 8192, 9973, 16384, 32768]


def _case(k):
    rng = np.random.default_rng(1000 + k)
    n = int(LENGTHS[k % len(LENGTHS)])
    dtype = np.complex128 if rng.random() < 0.5 else np.complex64
    if dtype == np.complex64 and n > 16384:
        dtype = np.complex128
    rows = int(rng.integers(1, 5))
    params = []
    for _ in range(rows):
        a = float(rng.uniform(-3, 3))
        b = float(rng.choice([-1, 1]) * 10 ** rng.uniform(-1.5, 1))
        d = float(rng.uniform(-3, 3))
        params.append((a, b, (a * d - 1.0) / b, d))
    abcd = np.array(params)
    f = ((rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))) / math.sqrt(2)).astype(dtype)
    return n, dtype, abcd, f


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    if not _t.cuda.is_available():
        pytest.skip("no CUDA device")
    return _t


@pytest.mark.parametrize("k", range(38))
def test_random_lct_rows(torch, k):
    from paper_0912_1379_b200 import ops

    n, dtype, abcd, f = _case(k)
    got = ops.lct_rows(torch.from_numpy(f).cuda(), abcd).cpu().numpy()
    _, ref = O.fast_lct_rows(abcd, f.astype(np.complex128))
    tol = 1e-12 if dtype == np.complex128 else 2e-5
    err = max_row_rel_l2(got.astype(np.complex128), ref)
    assert err <= tol, (n, dtype.__name__, abcd.tolist(), err)


@pytest.mark.parametrize("k", range(0, 38, 3))
def test_random_dft_rows(torch, k):
    from paper_0912_1379_b200 import ops

    n, dtype, _, f = _case(k)
    sign = -1 if k % 2 else 1
    got = ops.dft_rows(torch.from_numpy(f).cuda(), sign).cpu().numpy()
    ref = O.dft_rows(f.astype(np.complex128), sign)
    tol = 1e-12 if dtype == np.complex128 else 2e-5
    assert max_row_rel_l2(got.astype(np.complex128), ref) <= tol, (n, dtype.__name__)


# Batch sizes around the persistent grids of the row kernels that use split "buffer read" barriers and the
# L2 prefetch (c64 n = 16384: one CTA per SM; c128 n = 4096: two; c64 n = 1024: 8-row tiles): fewer rows than
# CTAs, one row more than a full round, ragged last tiles.  A row's result must not depend on the batch it is
# in (bitwise), must repeat bitwise, and must match the oracle.
@pytest.mark.parametrize("n,dtype,rows", [
    (16384, np.complex64, 1), (16384, np.complex64, 149), (16384, np.complex64, 300),
    (4096, np.complex128, 297), (4096, np.complex128, 593), (1024, np.complex64, 2371),
])
def test_persistent_grid_edges(torch, n, dtype, rows):
    from paper_0912_1379_b200 import ops

    rng = np.random.default_rng(n + rows)
    al = rng.uniform(0.05, np.pi - 0.05, rows)
    abcd = np.stack([np.cos(al), np.sin(al), -np.sin(al), np.cos(al)], 1)
    f = ((rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))) / math.sqrt(2)).astype(dtype)
    v = torch.from_numpy(f).cuda()
    got = ops.lct_rows(v, abcd).cpu().numpy()
    for _ in range(6 if n == 16384 else 2):  # (the split-barrier kernel: a shared-memory race would show up as jitter)
        again = ops.lct_rows(v, abcd).cpu().numpy()
        assert np.array_equal(got, again)
    pick = sorted({0, rows - 1, rows // 2, min(rows - 1, 148), min(rows - 1, 296)})
    for r in pick:  # the same row alone: another grid, another tile position
        alone = ops.lct_rows(v[r:r + 1].clone(), abcd[r:r + 1]).cpu().numpy()
        assert np.array_equal(alone[0], got[r]), (n, rows, r)
    _, ref = O.fast_lct_rows(abcd[pick], f[pick].astype(np.complex128))
    tol = 1e-12 if dtype == np.complex128 else 2e-5
    assert max_row_rel_l2(got[pick].astype(np.complex128), ref) <= tol
