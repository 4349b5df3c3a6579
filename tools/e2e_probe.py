"""Probe the host-buffer (end-to-end) path: pinned/pageable bandwidth and xft_lct_host timing."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0912_1379_b200 import ops, workloads  # noqa: E402

for dt in (np.complex64, np.complex128):
    c = workloads.config2(dtype=dt)
    hin = torch.from_numpy(c.values).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    print(dt.__name__, "pinned:", hin.is_pinned(), hout.is_pinned(), hin.nbytes >> 20, "MiB")
    d = hin.cuda()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        d.copy_(hin, non_blocking=True)
        hout.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    print("  torch H2D+D2H", f"{2 * 3 * hin.nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s")
    ops.lct_host(hin.numpy(), c.abcd, out=hout.numpy())
    for k in range(3):
        t = time.perf_counter()
        ops.lct_host(hin.numpy(), c.abcd, out=hout.numpy())
        dtm = time.perf_counter() - t
        print("  lct_host", f"{dtm * 1e3:.2f} ms", f"{2 * c.values.nbytes / dtm / 1e9:.1f} GB/s")
