"""2-D c64 LCT and column-pass timings over several shapes (K7 vs a variant library, e.g. -DXFT_COLRING=0).
XFT_LIB=tune/libxft_X.so python tools/time_2d_shapes.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from _variant import use_variant  # noqa: E402

tag = use_variant()
from paper_0912_1379_b200 import lct2d, workloads  # noqa: E402

p = np.array(workloads.CONFIG5_ABCD)


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for R, nc in ((4096, 4096), (8192, 8192), (4096, 16384), (16384, 2048), (32768, 4096), (65536, 2048), (16384, 16384)):
    f = torch.randn(R, nc, dtype=torch.complex64, device="cuda")
    full = f.clone()
    ws = torch.empty_like(full)
    out = torch.empty_like(full)
    tc = t(lambda: lct2d.columns_inplace(full, p, ws))
    try:
        t2 = t(lambda: lct2d.lct2d(f, p, p, out=out, workspace=ws))
    except Exception as e:  # rows longer than the row kernels take
        t2 = float("nan")
    gb = 2 * R * nc * 8 / 1e9
    print(f"{tag}: [{R} x {nc}] columns {tc:.3f} ms ({gb / tc:.0f} GB/s)   2-D {t2:.3f} ms", flush=True)
    del f, full, ws, out
