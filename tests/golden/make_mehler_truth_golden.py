"""Long-double evaluations of the dense Mehler formula for the golden cases with z = +-0.99
(tests/golden/golden.npz, n = 1024 and 4096), where the reference's own float64 formula loses
accuracy (catastrophic cancellation in (1+z^2)(x^2+y^2) - 4xyz near z = +-1).

    python tests/golden/make_mehler_truth_golden.py  ->  tests/golden/mehler_truth_golden.npz

Used by tests/test_gpu_chirpz.py::test_mehler_near_unit_z_against_long_double_truth: the GPU path is
held to 1e-12 against this truth, which is what justifies the 2e-12 bar against the reference's
own (less accurate) output for |1 - z^2| < 0.05.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import xft_oracle as O  # noqa: E402


def truth(z, f, n):
    x = O.asymptotic_nodes(n).astype(np.longdouble)
    dx = x[1] - x[0]
    zl = np.clongdouble(z)
    one = 1 - zl * zl
    a = np.sqrt(np.clongdouble(2) / one)
    fl = f.astype(np.clongdouble)
    g = np.empty(n, dtype=np.clongdouble)
    for j in range(n):
        expo = -((1 + zl * zl) * (x[j] * x[j] + x * x) - 4 * x[j] * x * zl) / (2 * one)
        g[j] = np.sum(a * np.exp(expo) * dx * fl)
    return g.astype(np.complex128)


def main():
    gold = np.load(os.path.join(HERE, "golden.npz"))
    out = {}
    for n in (1024, 4096):
        f = gold[f"mehler_in_n{n}"]
        for z in gold[f"mehler_z_n{n}"]:
            if abs(1 - z * z) < 0.05:
                key = f"n{n}_z{z.real:+.2f}"
                out[key + "_z"] = np.array([z])
                out[key] = truth(z, f, n)
                ref = gold[f"mehler_out_n{n}"][list(gold[f"mehler_z_n{n}"]).index(z)]
                print(key, "reference float64 vs long double:",
                      np.linalg.norm(ref - out[key]) / np.linalg.norm(out[key]))
    np.savez_compressed(os.path.join(HERE, "mehler_truth_golden.npz"), **out)


if __name__ == "__main__":
    main()
