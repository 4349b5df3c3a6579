"""CLI surface -- the parts that never touch the GPU.

Against the reference CLI's own output (tests/golden/cli_golden.json, made by
tests/golden/make_cli_golden.py running xft/cli.py): byte-identical grid CSVs
(asymptotic grid), and the exit codes of every malformed /
parameter-error invocation (xft/cli.py:378-397), which fail before any transform.
"""
import contextlib
import io
import json
import os
import tempfile

import numpy as np
import pytest

from paper_0912_1379_b200 import cli, hermite

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli_golden.json")))


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("name", ["grid8", "grid33"])
def test_grid_byte_identical(name):
    case = GOLD["cases"][name]
    rc, out, _ = run(case["argv"])
    assert rc == case["rc"] == 0
    assert out == case["stdout"]


@pytest.mark.parametrize("name", ["grid8_exact"])
def test_out_of_scope_requests_exit_2(name):
    """Exact Hermite zeros and the brute-force quadrature oracle are outside this build."""
    rc, out, err = run(GOLD["cases"][name]["argv"])
    assert rc == 2 and out == "" and err.startswith("error:")
    rc, out, err = run(["compare", "--n", "64", "--preset", "fourier", "--function", "gaussian:1,0,0",
                        "--oracle", "quadrature"])
    assert rc == 2 and err.startswith("error:")


@pytest.mark.parametrize("name", ["err_params", "err_unimodular", "err_both", "err_preset", "err_bzero_csv",
                                  "err_inverse_b"])
def test_error_exit_codes(name):
    case = GOLD["cases"][name]
    with tempfile.TemporaryDirectory() as tmp:
        g = hermite.asymptotic_zeros(8)
        with open(os.path.join(tmp, "in8.csv"), "w", encoding="utf-8", newline="\n") as f:
            f.write("x,re,im\n" + "".join(f"{float(x)!r},1,0\n" for x in g.nodes))
        rc, out, err = run([a.replace("{tmp}", tmp) for a in case["argv"]])
    assert rc == case["rc"]
    assert out == case["stdout"] == ""
    assert err.startswith("error:") or rc == 2


def test_usage_and_grid_errors(tmp_path):
    assert run(["nosuch"])[0] == 2
    assert run(["transform", "--n", "8"])[0] == 2                       # neither params nor preset
    assert run(["bench", "--sizes", ""])[0] == 2
    assert run(["bench", "--sizes", "8,x"])[0] == 2
    bad = tmp_path / "bad.csv"
    bad.write_text("t,re,im\n0,1,0\n")
    assert run(["transform", "--n", "1", "--preset", "fourier", "--input", str(bad)])[0] == 2   # header
    short = tmp_path / "short.csv"
    short.write_text("x,re,im\n0,1,0\n")
    rc, _, err = run(["transform", "--n", "8", "--preset", "fourier", "--input", str(short)])
    assert rc == 4 and "expected grid (k,x):" in err                    # grid mismatch prints the grid
    off = tmp_path / "off.csv"
    g = hermite.asymptotic_zeros(4)
    off.write_text("x,re,im\n" + "".join(f"{float(x) + 1e-6!r},1,0\n" for x in g.nodes))
    assert run(["transform", "--n", "4", "--preset", "fourier", "--input", str(off)])[0] == 4
