"""End-to-end (host buffers) config-2 step through xft_lct_host, the bench's two-thread form, through a
variant library: XFT_LIB=tune/libxft_X.so python tools/time_e2e.py [steps]"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

tag = use_variant()
import torch  # noqa: E402

from paper_0912_1379_b200 import ops, workloads  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
items = []
for dt in (np.complex64, np.complex128):
    c = workloads.config2(dtype=dt)
    hin = torch.from_numpy(c.values).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    items.append((hin, hout, c.abcd))


def step():
    ths = [threading.Thread(target=lambda a=a: (torch.cuda.set_device(0),
                                                 ops.lct_host(a[0].numpy(), a[2], out=a[1].numpy()))) for a in items]
    for t in ths:
        t.start()
    for t in ths:
        t.join()


step()
t0 = time.perf_counter()
for _ in range(steps):
    step()
dt = (time.perf_counter() - t0) / steps
print(f"{tag}: e2e step {dt * 1e3:.2f} ms, {2 * 4096 * 4096 / dt / 1e9:.3f} Gsamples/s")
