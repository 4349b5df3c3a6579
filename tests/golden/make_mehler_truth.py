"""Long-double evaluations of the dense Mehler formula (xft/dense.py:122-151) for the
config-3 rows where the reference's own float64 evaluation loses accuracy.

    python tests/golden/make_mehler_truth.py   ->  tests/golden/mehler_truth_cfg3.npz

g_j = sum_k sqrt(2/(1-z^2)) exp(-((1+z^2)(x_j^2+x_k^2) - 4 x_j x_k z) / (2(1-z^2))) dx f_k,
evaluated in numpy long double (x86 80-bit, 64-bit significand) on the same float64
nodes and inputs.  Used by tests/test_gpu_chirpz.py::test_mehler_config3_truth.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import xft_oracle as O  # noqa: E402
from paper_0912_1379_b200 import workloads  # noqa: E402

ROWS = (1013, 1, 382)  # z = -0.52i, -0.65i, -0.50i: unit-modulus kernels, large cancellation


def main():
    c3 = workloads.config3()
    z = c3.extra["z"]
    n = c3.values.shape[1]
    js = np.unique(np.concatenate([np.linspace(0, n - 1, 97).astype(int), n // 2 + np.arange(-40, 40, 7)]))
    x = O.asymptotic_nodes(n).astype(np.longdouble)
    dx = x[1] - x[0]
    out = {"js": js, "rows": np.array(ROWS)}
    for r in ROWS:
        zl = np.clongdouble(z[r])
        one = 1 - zl * zl
        a = np.sqrt(np.clongdouble(2) / one)
        f = c3.values[r].astype(np.clongdouble)
        g = np.empty(len(js), dtype=np.clongdouble)
        for i, j in enumerate(js):
            xj = x[j]
            expo = -((1 + zl * zl) * (xj * xj + x * x) - 4 * xj * x * zl) / (2 * one)
            g[i] = np.sum(a * np.exp(expo) * dx * f)
        out[f"truth_{r}"] = g.astype(np.complex128)
        ref = O.mehler_apply(z[r], c3.values[r], rows_out=js)
        print(r, z[r], "float64 dense formula vs long double:",
              np.linalg.norm(ref - out[f"truth_{r}"]) / np.linalg.norm(out[f"truth_{r}"]))
    np.savez_compressed(os.path.join(HERE, "mehler_truth_cfg3.npz"), **out)


if __name__ == "__main__":
    main()
