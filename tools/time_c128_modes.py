"""c128 4096 x 4096 row kernel by chirp mode mix: config 2's angles (81% smooth walk, 19% corrected), all rows
smooth (alpha = 1.0), all rows corrected (alpha = 0.1).  Shows what the static row assignment loses to the mix."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0912_1379_b200 import ops, workloads  # noqa: E402

c = workloads.config2(dtype=np.complex128)
v = [torch.from_numpy(c.values).cuda() for _ in range(3)]
o = [torch.empty_like(x) for x in v]


def run(abcd, reps=20):
    p = torch.from_numpy(np.ascontiguousarray(abcd)).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            ops.lct_rows(v[i], p, out=o[i], validate=False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            ops.lct_rows(v[i % 3], p, out=o[i % 3], validate=False)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def frft(al):
    return np.stack([np.cos(al), np.sin(al), -np.sin(al), np.cos(al)], 1)


rows = c.values.shape[0]
print("config-2 mix      %.2f us" % run(c.abcd))
print("all smooth walk   %.2f us" % run(frft(np.full(rows, 1.0))))
print("all corrected     %.2f us" % run(frft(np.full(rows, 0.1))))
al = np.sort(np.arccos(c.abcd[:, 0]))  # the same angles sorted: like modes adjacent
print("mix, sorted rows  %.2f us" % run(frft(al)))
