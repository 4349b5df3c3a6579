import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_0912_1379_b200 import ops
for n, B in ((512, 131072), (2048, 32768), (1024, 65536)):
    v = torch.randn(B, n, dtype=torch.complex64, device="cuda")
    o = torch.empty_like(v)
    p = np.array([0.3, 1.1, -0.7, 0.77 + 0.7 * 0.3 / 1.1 * 0 + 0.0])
    p = np.array([0.0, 1.0, -1.0, 0.0])
    for _ in range(3): ops.lct_rows(v, p, out=o)
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ops.lct_rows(v, p, out=o)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(n, f"{ms*1e3:.1f} us", f"{16 * B * n / ms / 1e6:.0f} GB/s")
