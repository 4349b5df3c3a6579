"""Column-pass timing: one [16384, 16384] c64 field vs 8 slabs of [16384, 2048] (the sharded layout)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0912_1379_b200 import lct2d, workloads

p = np.array(workloads.CONFIG5_ABCD)
n = 16384


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = torch.randn(n, n, dtype=torch.complex64, device="cuda")
ws = torch.empty_like(full)
print("full field columns", t(lambda: lct2d.columns_inplace(full, p, ws)), "ms")
for G in (2, 4, 8):
    slabs = [torch.randn(n, n // G, dtype=torch.complex64, device="cuda") for _ in range(G)]
    wss = [torch.empty_like(s) for s in slabs]
    print(f"{G} slabs [{n}, {n // G}] columns", t(lambda: [lct2d.columns_inplace(s, p, w) for s, w in zip(slabs, wss)]), "ms")
