"""Config-3 Mehler step, graph-replayed over 3 rotating buffer sets (the bench's method), through a
variant library: XFT_LIB=tune/libxft_X.so python tools/time_cfg3.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

tag = use_variant()
import torch  # noqa: E402

from paper_0912_1379_b200 import mehler, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = workloads.config3()
z = c.extra["z"]
sets = [(torch.from_numpy(c.values).cuda(), None) for _ in range(3)]
sets = [(v, torch.empty_like(v)) for v, _ in sets]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for v, o in sets:
        mehler.mehler_rows(v, z, out=o)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            v, o = sets[i % 3]
            mehler.mehler_rows(v, z, out=o)
g.replay()
torch.cuda.synchronize()
best = 1e9
with torch.cuda.stream(s):  # replay on the stream the events are recorded on
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
print(f"{tag}: cfg3 {best:.4f} ms per step")
