"""Golden outputs of the reference CLI and oracles.

Run in the build container only (imports /root/reference/pkg/src/xft):

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli_golden.json: the reference CLI's exact stdout/CSV text
and exit codes for a set of invocations, plus oracle values (closed form,
quadrature, dense LCT / scaled Fourier / Mehler entries) at small sizes.
"""
from __future__ import annotations

import contextlib
import io
import json
import math
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import xft  # noqa: E402  (the reference)
from xft import cli as rcli  # noqa: E402
from xft import dense as rdense  # noqa: E402
from xft import kernel as rkernel  # noqa: E402
from xft import oracle as roracle  # noqa: E402

# invocations; "{tmp}" is replaced by a scratch directory; output file text is captured
CASES = {
    "grid8": ["grid", "--n", "8"],
    "grid33": ["grid", "--n", "33"],
    "grid8_exact": ["grid", "--n", "8", "--exact"],
    "grid33_exact": ["grid", "--n", "33", "--exact"],
    "transform_cfg1ish": ["transform", "--n", "64", "--params", "2,1,1,1", "--function", "gaussian:1,0.2,0.1"],
    "transform_fourier": ["transform", "--n", "32", "--preset", "fourier", "--function", "gaussian:1,0,0"],
    "transform_frft": ["transform", "--n", "128", "--preset", "frft:0.7", "--function", "gaussian:0.5,0.1,0"],
    "transform_bzero": ["transform", "--n", "16", "--params", "0.5,0,1.5,2", "--function", "gaussian:1,0.3,0"],
    "compare_closed": ["compare", "--n", "256", "--preset", "frft:0.4", "--function", "gaussian:1,0.2,0.1",
                       "--max-abs", "1e-9"],
    "compare_dense": ["compare", "--n", "64", "--params", "1,2,0.5,2", "--function", "gaussian:1,0.3,0.1",
                      "--oracle", "dense"],
    "compare_quad": ["compare", "--n", "64", "--preset", "fourier", "--function", "gaussian:1,0,0",
                     "--oracle", "quadrature"],
    "compare_inverse": ["compare", "--n", "256", "--params", "1,2,0.5,2", "--function", "gaussian:1,0.3,0.1",
                        "--inverse", "--max-abs", "1e-10"],
    "compare_threshold": ["compare", "--n", "64", "--preset", "fourier", "--function", "gaussian:1,0,0",
                          "--max-abs", "1e-30"],
    "err_inverse_b": ["compare", "--n", "32", "--params", "1,-2,0.5,-2.25", "--no-unimodular-check",
                      "--function", "gaussian:1,0,0", "--inverse"],
    "err_params": ["transform", "--n", "8", "--params", "1,2,3"],
    "err_unimodular": ["transform", "--n", "8", "--params", "1,2,3,4", "--function", "gaussian:1,0,0"],
    "err_both": ["transform", "--n", "8", "--preset", "fourier"],
    "err_preset": ["transform", "--n", "8", "--preset", "nope", "--function", "gaussian:1,0,0"],
    "err_bzero_csv": ["transform", "--n", "8", "--params", "1,0,0,1", "--input", "{tmp}/in8.csv"],
}


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = rcli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def main():
    res = {"cases": {}, "oracles": {}}
    with tempfile.TemporaryDirectory() as tmp:
        g = xft.asymptotic_zeros(8)
        with open(os.path.join(tmp, "in8.csv"), "w", encoding="utf-8", newline="\n") as f:
            f.write("x,re,im\n" + "".join(f"{float(x)!r},1,0\n" for x in g.nodes))
        for name, argv in CASES.items():
            argv = [a.replace("{tmp}", tmp) for a in argv]
            rc, so, se = run(argv)
            res["cases"][name] = {"argv": CASES[name], "rc": rc, "stdout": so}
    # oracle values
    gp = roracle.GaussianParams(1.0, 0.25, 0.1)
    p = xft.LctParams(0.5, 1.5, -0.5, 0.5)
    ys = np.linspace(-3, 3, 13)
    res["oracles"]["closed_form"] = {"g": [1.0, 0.25, 0.1], "abcd": list(p.as_tuple()), "y": ys.tolist(),
                                     "re": np.real(roracle.gaussian_lct_closed_form(gp, p, ys)).tolist(),
                                     "im": np.imag(roracle.gaussian_lct_closed_form(gp, p, ys)).tolist()}
    qv = roracle.quadrature_on_nodes(p, gp.evaluate, ys, roracle.QuadratureConfig(radius=12.0, tol=1e-10))
    res["oracles"]["quadrature"] = {"re": np.real(qv).tolist(), "im": np.imag(qv).tolist()}
    n = 48
    for name, mat in (("F", rkernel.scaled_fourier_matrix(n)), ("L", rdense.dense_lct_matrix(n, p).entries),
                      ("mehler", rdense.frft_matrix_asymptotic(n, rdense.FrftOrder(0.3 + 0.6j)).entries)):
        res["oracles"][f"dense_{name}"] = {"n": n, "re": np.real(mat).ravel().tolist(),
                                          "im": np.imag(mat).ravel().tolist()}
    path = os.path.join(HERE, "cli_golden.json")
    with open(path, "w", encoding="utf-8") as f:
        json.dump(res, f)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
