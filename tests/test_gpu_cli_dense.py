"""GPU tests of the CLI transforms and the dense oracles.

* CLI: every transform/compare case of tests/golden/cli_golden.json (the
  reference CLI's own output): same exit code, same header, byte-identical
  abscissa column, values within the c128 tolerance; compare reports under the
  reference tests' thresholds (pkg/tests/test_cli.py:160-183).
* Dense oracles: GPU entries of F, L and K_z dx against the reference's
  matrices (xft/kernel.py:68-80, xft/dense.py:122-151, 230-249); matrix-free
  dense products against the oracle and against the fast kernels at full size.
* The CLI's Gaussian closed form against the reference's closed form and quadrature values.
"""
import contextlib
import io
import json
import math
import os

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import max_row_rel_l2, rel_l2

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli_golden.json")))


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


def run(argv):
    from paper_0912_1379_b200 import cli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def table(text):
    lines = text.strip("\n").split("\n")
    return lines[0], [ln.split(",") for ln in lines[1:]]


@pytest.mark.parametrize("name", ["transform_cfg1ish", "transform_fourier", "transform_frft", "transform_bzero"])
def test_cli_transform_matches_reference(torch, name):
    case = GOLD["cases"][name]
    rc, out, _ = run(case["argv"])
    assert rc == case["rc"] == 0
    h1, r1 = table(out)
    h0, r0 = table(case["stdout"])
    assert h1 == h0 == "y,re,im" and len(r1) == len(r0)
    assert [r[0] for r in r1] == [r[0] for r in r0]          # output nodes byte-identical
    got = np.array([[float(r[1]), float(r[2])] for r in r1])
    ref = np.array([[float(r[1]), float(r[2])] for r in r0])
    gc, rc_ = got[:, 0] + 1j * got[:, 1], ref[:, 0] + 1j * ref[:, 1]
    assert rel_l2(gc, rc_) <= 1e-12
    for r in r1:                                              # 17 significant digits (lossless)
        for v in r:
            assert float(format(float(v), ".17g")) == float(v)


@pytest.mark.parametrize("name", ["compare_closed", "compare_dense", "compare_inverse", "compare_threshold"])
def test_cli_compare_matches_reference(torch, name):
    case = GOLD["cases"][name]
    rc, out, _ = run(case["argv"])
    assert rc == case["rc"]
    lines, ref_lines = out.strip().split("\n"), case["stdout"].strip().split("\n")
    assert lines[0] == ref_lines[0] and len(lines) == len(ref_lines)   # header + rows + report line
    assert [ln.split(",")[0] for ln in lines[1:-1]] == [ln.split(",")[0] for ln in ref_lines[1:-1]]
    n, max_abs, rms, rel = lines[-1].split(",")
    assert int(n) == int(ref_lines[-1].split(",")[0])
    assert float(max_abs) <= max(1e-10, 10 * float(ref_lines[-1].split(",")[1]))


def test_cli_csv_roundtrip_and_bench(torch, tmp_path):
    src = tmp_path / "in.csv"
    rc, out, _ = run(["grid", "--n", "64"])
    xs = [float(ln.split(",")[1]) for ln in out.strip().split("\n")[1:]]
    src.write_text("x,re,im\n" + "".join(f"{x!r},{math.exp(-x * x / 2)!r},0\n" for x in xs))
    rc, a, _ = run(["transform", "--n", "64", "--preset", "fourier", "--input", str(src)])
    rc2, b, _ = run(["transform", "--n", "64", "--preset", "fourier", "--function", "gaussian:0.5,0,0"])
    assert rc == rc2 == 0
    ta, tb = table(a)[1], table(b)[1]
    va = np.array([complex(float(r[1]), float(r[2])) for r in ta])
    vb = np.array([complex(float(r[1]), float(r[2])) for r in tb])
    assert [r[0] for r in ta] == [r[0] for r in tb] and rel_l2(va, vb) <= 1e-14
    outp = tmp_path / "bench.tsv"
    assert run(["bench", "--sizes", "64,128", "--repeats", "2", "--output", str(outp)])[0] == 0
    lines = outp.read_text().split("\n")
    assert lines[0] == "n\tseconds\tratio_vs_half" and lines[1].startswith("64\t") and lines[2].startswith("128\t")


def _gold_matrix(key):
    d = GOLD["oracles"][key]
    n = d["n"]
    return n, (np.array(d["re"]) + 1j * np.array(d["im"])).reshape(n, n)


def test_dense_entries_match_reference(torch, X):
    from paper_0912_1379_b200 import dense

    n, F = _gold_matrix("dense_F")
    assert rel_l2(dense.scaled_fourier_matrix_gpu(n), F) <= 1e-14
    _, L = _gold_matrix("dense_L")
    p = tuple(GOLD["oracles"]["closed_form"]["abcd"])
    assert rel_l2(dense.dense_lct_matrix(n, X.LctParams(*p)).entries, L) <= 1e-14
    _, K = _gold_matrix("dense_mehler")
    assert rel_l2(X.frft_matrix_asymptotic(n, X.FrftOrder(0.3 + 0.6j)).entries, K) <= 1e-14
    with pytest.raises(X.errors.InvalidSizeError):
        dense.dense_entries(4097, dense.KIND_F)


@pytest.mark.parametrize("n", [37, 256, 1000, 4096])
def test_dense_lct_apply_vs_oracle_and_fast(torch, X, n):
    from paper_0912_1379_b200 import dense, ops

    rng = np.random.default_rng(n)
    f = rng.normal(size=(3, n)) + 1j * rng.normal(size=(3, n))
    p = (0.5, 1.5, -0.5, 0.5)
    got = dense.dense_lct_apply(f, p).cpu().numpy()
    _, ref = O.fast_lct_rows(p, f)                            # oracle: the reference algorithm
    assert max_row_rel_l2(got, ref) <= 1e-12
    Fv = dense.dense_lct_apply(f, None).cpu().numpy()        # scaled Fourier matrix
    assert max_row_rel_l2(Fv, O.scaled_fourier_rows(f)) <= 1e-12
    if n == 4096:                                             # independent check of the fast GPU path
        fast = ops.lct_rows(torch.from_numpy(f).cuda(), p).cpu().numpy()
        assert max_row_rel_l2(fast, got) <= 1e-12


def test_dense_mehler_full_size_rows(torch, X):
    """Config-3 rows at n = 16384 with the O(n^2) dense product vs the fast windowed kernel."""
    from paper_0912_1379_b200 import dense, workloads

    c = workloads.config3(rows=6)
    v = torch.from_numpy(c.values).cuda()
    z = c.extra["z"]
    fast = X.mehler_rows(v, z).cpu().numpy()
    slow = dense.dense_mehler_apply(v, z).cpu().numpy()
    zz = np.asarray(z).reshape(-1)
    for r in range(v.shape[0]):
        tol = 2e-12 if abs(1 - zz[r] ** 2) < 0.05 else 1e-12
        assert rel_l2(fast[r], slow[r]) <= tol * 10
    # and against the oracle's chunked dense restatement at a smaller size
    rng = np.random.default_rng(3)
    f = rng.normal(size=2048) + 1j * rng.normal(size=2048)
    g = dense.dense_mehler_apply(f, 0.6 + 0.3j)[0].cpu().numpy()
    assert rel_l2(g, O.mehler_apply(0.6 + 0.3j, f)) <= 1e-12


def test_closed_form_matches_reference_oracles():
    """The CLI's completed-square Gaussian closed form vs the reference's own closed form and its
    brute-force quadrature values (tests/golden/cli_golden.json, xft/oracle.py)."""
    from paper_0912_1379_b200 import cli
    from paper_0912_1379_b200.lct import LctParams

    d = GOLD["oracles"]["closed_form"]
    ys = np.array(d["y"])
    cf = cli.gaussian_closed_form(cli.Gaussian(*d["g"]), LctParams(*d["abcd"]), ys)
    ref_cf = np.array(d["re"]) + 1j * np.array(d["im"])
    ref_q = np.array(GOLD["oracles"]["quadrature"]["re"]) + 1j * np.array(GOLD["oracles"]["quadrature"]["im"])
    assert np.max(np.abs(cf - ref_cf)) <= 1e-14 * np.max(np.abs(ref_cf))
    assert np.max(np.abs(cf - ref_q)) <= 1e-12
