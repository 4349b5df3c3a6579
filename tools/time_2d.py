"""Time the single-GPU 2-D LCT of config 5 (and its two phases)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0912_1379_b200 import lct2d, ops, workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
f = torch.from_numpy(workloads.config5_field(n)).cuda()
out, ws = torch.empty_like(f), torch.empty_like(f)
p = np.array(workloads.CONFIG5_ABCD)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print("rows", t(lambda: ops.lct_rows(f, p, out=out, validate=False)), "ms")
print("cols", t(lambda: lct2d.columns_inplace(out, p, ws)), "ms")
print("2d", t(lambda: lct2d.lct2d(f, p, p, out=out, workspace=ws)), "ms")
