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
