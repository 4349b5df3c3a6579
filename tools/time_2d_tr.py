"""Time config 5 as two row passes with transposed (column-scatter) stores vs the current lct2d."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0912_1379_b200 import _native, lct2d, ops, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
f = torch.from_numpy(workloads.config5_field(n)).cuda()
out, ws, out2 = torch.empty_like(f), torch.empty_like(f), torch.empty_like(f)
p = np.ascontiguousarray(np.array(workloads.CONFIG5_ABCD, dtype=np.float64))


def rows_t(src, dst):
    _native.call("xft_lct_rows_packed", src.data_ptr(), dst.data_ptr(), n, n, ops._dtype_code(src), p.ctypes.data,
                 0, n, ops._stream_ptr(src.device))


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


print("rows natural", t(lambda: ops.lct_rows(f, p, out=out, validate=False)), "ms")
print("rows transposed store", t(lambda: rows_t(f, ws)), "ms")
print("2d current", t(lambda: lct2d.lct2d(f, p, p, out=out, workspace=ws)), "ms")
print("2d two transposed row passes", t(lambda: (rows_t(f, ws), rows_t(ws, out2))), "ms")
lct2d.lct2d(f, p, p, out=out, workspace=ws)
rows_t(f, ws)
rows_t(ws, out2)
torch.cuda.synchronize()
d = (out2 - out).abs().pow(2).sum().sqrt() / out.abs().pow(2).sum().sqrt()
print("rel diff", float(d))
