"""Writes tests/golden/hermite_rows.npz: the reference's own hermite_function_row outputs.

Runs the reference (``/root/reference/pkg/src/xft``, xft/hermite.py:92-112) at
the points the configs use -- every node of the n=1024 grid, a strided sample
of the n=16384 grid (config 3, psi_0..30) and a few off-grid points -- so the
package's vectorised ``hermite_function_table`` (which generates the config-3
and config-4 inputs) is pinned to the reference bit for bit
(tests/test_oracle.py::test_hermite_table_matches_reference_rows).
Re-run only where /root/reference exists:  python tests/golden/make_hermite_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import xft  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    x1024 = xft.asymptotic_zeros(1024).nodes
    x16384 = xft.asymptotic_zeros(16384).nodes[::97]
    extra = np.array([0.0, 1e-300, -0.5, 3.25, 12.0, -37.5, 141.0])
    out = {}
    for name, xs, m in (("n1024_m21", x1024, 21), ("n16384_m31", x16384, 31), ("extra_m40", extra, 40)):
        out[f"{name}_x"] = xs
        out[f"{name}_psi"] = np.stack([xft.hermite_function_row(m, float(x)) for x in xs], axis=1)
    np.savez_compressed(os.path.join(HERE, "hermite_rows.npz"), **out)


if __name__ == "__main__":
    main()
