"""Per-row c128 error of config 2 against the oracle on the rows whose largest input phase lies in a band.

  XFT_LIB=... python tools/c128_rowerr.py [lo hi]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

use_variant()
import torch

from oracle import xft_oracle as O
from paper_0912_1379_b200 import ops, workloads

lo, hi = (float(sys.argv[1]), float(sys.argv[2])) if len(sys.argv) > 2 else (2048.0, 4096.0)
c2 = workloads.config2(dtype=np.complex128)
n = 4096
half = (np.pi / np.sqrt(2 * n)) / 2
xm = (n - 1) * half
a, b = c2.abcd[:, 0], c2.abcd[:, 1]
pin = np.abs(0.5 * a / b) * xm * xm
rows = np.where((pin >= lo) & (pin < hi))[0]
rows = rows[np.linspace(0, len(rows) - 1, min(24, len(rows))).astype(int)]
got = ops.lct_rows(torch.from_numpy(c2.values[rows]).cuda(), c2.abcd[rows]).cpu().numpy()
_, ref = O.fast_lct_rows(c2.abcd[rows], c2.values[rows])
err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
print(f"band [{lo}, {hi}): {len(rows)} rows, max rel_l2 {err.max():.3e}, mean {err.mean():.3e}")
