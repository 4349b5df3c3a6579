"""Column pass alone on a 16384^2 c64 field (K7 vs whatever XFT_LIB builds), plus the full 2-D step.
python tools/time_colring.py [n]"""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384


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


torch.manual_seed(7)
f = torch.randn(n, n, dtype=torch.complex64, device="cuda")
full = f.clone()
ws = torch.empty_like(full)
out = torch.empty_like(full)
print(f"{tag}: columns in place {n}^2: {t(lambda: lct2d.columns_inplace(full, p, ws)):.3f} ms", flush=True)
print(f"{tag}: 2-D {n}^2: {t(lambda: lct2d.lct2d(f, p, p, out=out, workspace=ws)):.3f} ms", flush=True)
import hashlib  # noqa: E402

lct2d.lct2d(f, p, p, out=out, workspace=ws)
torch.cuda.synchronize()
print(f"{tag}: 2-D output sha {hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]}", flush=True)
