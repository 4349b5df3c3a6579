"""GPU Mehler rows vs a long-double evaluation of the dense formula (truth files from the host)."""
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
for r in (1013, 1):
    t = np.load(os.path.join(sys.argv[1], f"truth_{r}.npy"))
    js = t[0].astype(int)
    truth = t[1] + 1j * t[2]
    ref = O.mehler_apply(z[r], c3.values[r], rows_out=js)
    rl = lambda a: np.linalg.norm(a - truth) / np.linalg.norm(truth)
    print(r, f"gpu vs truth {rl(got[r, js]):.3e}  oracle vs truth {rl(ref):.3e}  gpu vs oracle "
             f"{np.linalg.norm(got[r, js] - ref) / np.linalg.norm(ref):.3e}")
