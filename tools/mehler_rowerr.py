"""Config-3 Mehler rows of test_mehler_config3_full: error against the dense oracle per row."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from oracle import xft_oracle as O
from paper_0912_1379_b200 import mehler, workloads

c3 = workloads.config3()
z = c3.extra["z"]
got = mehler.mehler_rows(torch.from_numpy(c3.values).cuda(), z).cpu().numpy()
n = 16384
gam = np.where((2 * z / (1 - z * z)).real >= 0, (1 - z) / (2 * (1 + z)), (1 + z) / (2 * (1 - z))).real
rows = list(np.argsort(gam)[:4]) + list(np.argsort(gam)[-2:]) + [0, 1, 511]
js = np.linspace(0, n - 1, 97).astype(int)
js = np.unique(np.concatenate([js, n // 2 + np.arange(-40, 40, 7)]))
for r in rows:
    ref = O.mehler_apply(z[r], c3.values[r], rows_out=js)
    e = np.linalg.norm(got[r, js] - ref) / np.linalg.norm(ref)
    print(r, z[r], f"{e:.3e}", flush=True)
