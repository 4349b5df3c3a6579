"""CPU-side checks of the native library and host logic (no GPU compute)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_0912_1379_b200 import _native, errors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib_or_skip():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libxft_b200.so not built (run __graft_entry__.build())")
    return _native.load_library()


def test_header_symbols_exported():
    lib = _lib_or_skip()
    header = open(os.path.join(ROOT, "include", "xft_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t)\s+(xft_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.EXPORTED)


def test_version_and_limits():
    lib = _lib_or_skip()
    assert lib.xft_version() >= 100
    assert lib.xft_max_n(0) >= 16384
    assert lib.xft_max_n(1) >= 8192


def _validate(lib, P, check=1, tol=1e-10):
    P = np.ascontiguousarray(P, dtype=np.float64)
    bad = ctypes.c_int64(-1)
    st = lib.xft_validate_lct_params(P.ctypes.data, P.reshape(-1, 4).shape[0], 4, check, tol, ctypes.byref(bad))
    return st, bad.value


def test_param_validation_order():
    lib = _lib_or_skip()
    ok = np.array([[0.0, 1.0, -1.0, 0.0], [1.0, 2.0, 0.5, 2.0]])
    assert _validate(lib, ok) == (0, -1)
    # b == 0 anywhere wins over a non-unimodular earlier row (reference checks b first)
    P = np.array([[1.0, 1.0, 1.0, 1.0], [1.0, 0.0, 0.0, 1.0]])
    assert _validate(lib, P) == (4, 1)
    P = np.array([[0.0, 1.0, -1.0, 0.0], [1.0, 1.0, 1.0, 1.0]])
    assert _validate(lib, P) == (2, 1)
    assert _validate(lib, P, check=0) == (0, -1)
    # unimodular tolerance: 5e-11 off passes (pkg/tests/test_lct.py:56-60)
    assert _validate(lib, np.array([[1.0, 1.0, 1.0, 2 + 5e-11]]))[0] == 0
    assert _validate(lib, np.array([[np.nan, 1.0, 1.0, 1.0]]))[0] == 2


def test_mehler_z_validation():
    lib = _lib_or_skip()
    bad = ctypes.c_int64(-1)
    for z, code in [((0.5, 0.0), 0), ((1.0, 0.0), 3), ((-1.0, 0.0), 3), ((0.0, 1.0), 0), ((1.1, 0.0), 2)]:
        a = np.array(z, dtype=np.float64)
        assert lib.xft_validate_mehler_z(a.ctypes.data, 1, 2, ctypes.byref(bad)) == code, z


def test_b_zero_validation_order():
    """xft/lct.py:243-253: b != 0, then a*d = 1, then d > 0; per-row bad index."""
    lib = _lib_or_skip()
    bad = ctypes.c_int64(-1)

    def v(P, stride=4):
        P = np.ascontiguousarray(P, dtype=np.float64)
        bad.value = -1
        return lib.xft_validate_b_zero(P.ctypes.data, P.reshape(-1, 4).shape[0], stride, 1e-10, ctypes.byref(bad)), \
            bad.value

    assert v([[1.0, 0.0, 3.0, 1.0], [0.5, 0.0, 0.0, 2.0]]) == (0, -1)
    assert v([[1.0, 0.0, 3.0, 1.0], [0.0, 1.0, -1.0, 0.0]]) == (2, 1)     # b != 0
    assert v([[1.0, 0.0, 3.0, 1.0], [1.0, 0.0, 0.0, 2.0]]) == (2, 1)     # a d != 1
    assert v([[-1.0, 0.0, 0.0, -1.0]]) == (5, 0)                         # d <= 0
    assert v([[-1.0, 1.0, 0.0, -1.0]]) == (2, 0)                         # b checked first
    assert v([[0.5, 0.0, 0.0, 2.0]], stride=0) == (0, -1)


def test_status_mapping():
    with pytest.raises(errors.DegenerateParameterError):
        errors.raise_for(4, "x")
    with pytest.raises(errors.GridMismatchError):
        errors.raise_for(7, "x")
    assert issubclass(errors.GridMismatchError, errors.ShapeError)
    assert issubclass(errors.SingularParameterError, errors.ParameterError)
    errors.raise_for(0, "ok")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_0912_1379_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def test_no_cuda_means_loud_failure(monkeypatch):
    import torch

    import paper_0912_1379_b200 as X

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeUnavailable):
        X.fast_lct(X.LctParams.fourier(), X.Signal(X.asymptotic_zeros(8), np.ones(8)))


@pytest.mark.parametrize("R,ncols", [(16384, 16384), (16384, 24), (16384, 2048), (32768, 528), (32768, 40),
                                     (65536, 200), (16384, 64 * 7)])
def test_column_ring_schedule_is_deadlock_free(R, ncols):
    """The tile order of the L2-staged column kernel (xft_colring.cuh): every (pass, block, line) once,
    and each tile's dependencies carry smaller indices -- pass 2 of a super-block after all of its
    pass-1 tiles, pass 1 of super-block s after every pass-2 tile of s - slots (the ring slot it
    overwrites).  With CTA b running tiles b, b + grid, ... in order on a cooperative (all-resident)
    grid, the lowest unfinished tile can then always run."""
    lib = _lib_or_skip()
    info = (ctypes.c_int * 6)()
    tile = (ctypes.c_int * 5)()
    assert lib.xft_column_schedule(R, ncols, 0, tile, info) == 0
    total, nsb, lag, slots, t0, t1 = list(info)
    assert 1 <= lag <= nsb and 1 <= slots <= nsb and total == nsb * (t0 + t1)
    seen = set()
    last_p1 = {}   # super-block -> largest pass-1 index
    first_p2 = {}  # super-block -> smallest pass-2 index
    last_p2 = {}
    first_p1 = {}
    count = {}
    for i in range(total):  # every tile: the decode is host code, microseconds each
        assert lib.xft_column_schedule(R, ncols, i, tile, None) == 0
        ph, sb, cb, idx, slot = list(tile)
        assert ph in (0, 1) and 0 <= sb < nsb and slot == sb % slots
        key = (ph, cb, idx)
        assert key not in seen
        seen.add(key)
        count[(ph, sb)] = count.get((ph, sb), 0) + 1
        if ph == 0:
            last_p1[sb] = i
            first_p1.setdefault(sb, i)
        else:
            first_p2.setdefault(sb, i)
            last_p2[sb] = i
    assert lib.xft_column_schedule(R, ncols, total, tile, None) == 0 and tile[0] == 2
    for sb in range(nsb):
        assert count[(0, sb)] == t0 and count[(1, sb)] == t1
        assert last_p1[sb] < first_p2[sb]
        if sb >= slots:
            assert last_p2[sb - slots] < first_p1[sb]


def test_column_ring_schedule_rejects_other_shapes():
    lib = _lib_or_skip()
    for R, nc in ((2048, 64), (8192, 64), (1 << 17, 64), (20000, 64), (16384, 0)):
        assert lib.xft_column_schedule(R, nc, 0, None, None) != 0
