"""One single-GPU 2-D LCT of a random 16384^2 c64 field on the device (ncu captures of the row and
cluster column kernels without the host-side field generation).  python tools/prof_2d.py [reps] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0912_1379_b200 import lct2d, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
f = torch.randn(n, n, dtype=torch.complex64, device="cuda")
out, ws = torch.empty_like(f), torch.empty_like(f)
for _ in range(reps):
    lct2d.lct2d(f, workloads.CONFIG5_ABCD, workloads.CONFIG5_ABCD, out=out, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    lct2d.lct2d(f, workloads.CONFIG5_ABCD, workloads.CONFIG5_ABCD, out=out, workspace=ws)
e1.record()
torch.cuda.synchronize()
print(f"2-D {n}^2 c64: {e0.elapsed_time(e1) / reps:.3f} ms per transform")
