"""Accuracy probe: the reference's acceptance criteria 2/3 (figure-1 / figure-2 configurations,
central-80% max-abs error of fast_lct vs the reference's direct quadrature) for the GPU path,
beside the reference's own fast_lct error.  XFT_LIB=variant.so python tools/fig_err.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

tag = use_variant()
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import xft as R  # noqa: E402  (the reference, for the oracle and its own error)
import xft.calibration  # noqa: E402,F401

from paper_0912_1379_b200 import lct as L  # noqa: E402
from paper_0912_1379_b200.hermite import asymptotic_zeros  # noqa: E402

out = {"tag": tag}
for name, g, p, n in (("fig1", R.calibration.FIGURE1_GAUSSIAN, R.calibration.FIGURE1_PARAMS, R.calibration.FIGURE1_N),
                      ("fig2", R.calibration.FIGURE2_GAUSSIAN, R.calibration.FIGURE2_PARAMS, R.calibration.FIGURE2_N)):
    grid = asymptotic_zeros(n)
    f = g.evaluate(grid.nodes).astype(complex)
    ours = L.fast_lct(L.LctParams(*p.as_tuple()), L.Signal(grid, f))
    ref = R.fast_lct(p, R.Signal(R.asymptotic_zeros(n), f))
    sl = slice(n // 10, (9 * n) // 10)
    q = R.quadrature_on_nodes(p, g.evaluate, ref.output_nodes[sl], R.QuadratureConfig.for_gaussian(g), threads=1)
    out[name] = {"ours": float(np.max(np.abs(ours.values[sl] - q))), "reference": float(np.max(np.abs(ref.values[sl] - q))),
                 "ours_vs_ref_rel": float(np.linalg.norm(ours.values - ref.values) / np.linalg.norm(ref.values))}
print(json.dumps(out), flush=True)
