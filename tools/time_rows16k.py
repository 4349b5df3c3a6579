"""Row pass of config 5 alone: 16384 rows x 16384 c64, (1,0.25,0,1), graph-replayed over 2 buffer
sets.  XFT_LIB=tune/libxft_X.so python tools/time_rows16k.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

tag = use_variant()
import torch  # noqa: E402

from paper_0912_1379_b200 import ops  # noqa: E402

n = 16384
sets = [torch.randn(n, n, dtype=torch.complex64, device="cuda") for _ in range(2)]
outs = [torch.empty_like(v) for v in sets]
p = torch.tensor([1.0, 0.25, 0.0, 1.0], dtype=torch.float64, device="cuda")  # device params: capturable
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for v, o in zip(sets, outs):
        ops.lct_rows(v, p, out=o, validate=False)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(6):
            ops.lct_rows(sets[i % 2], p, out=outs[i % 2], validate=False)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 6)
gb = 2 * n * n * 8 / 1e9
print(f"{tag}: rows 16384^2 c64 {best * 1e3:.1f} us, {gb / (best * 1e-3):.0f} GB/s")
