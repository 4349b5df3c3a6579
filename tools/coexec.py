"""Tuning experiment: c64 and c128 cfg2 batches on two streams with capped persistent grids.

  XFT_LIB=tune/libxft_cap.so python tools/coexec.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

use_variant()


def main():
    import torch

    from paper_0912_1379_b200 import ops, workloads

    c64 = workloads.config2(dtype=np.complex64)
    c128 = workloads.config2(dtype=np.complex128)
    data = {}
    for tag, c in (("c64", c64), ("c128", c128)):
        v = torch.from_numpy(c.values).cuda()
        data[tag] = (v, torch.empty_like(v), torch.from_numpy(c.abcd).cuda())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(tag, st):
        v, o, p = data[tag]
        with torch.cuda.stream(st):
            ops.lct_rows(v, p, out=o, validate=False)

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
        return round(best, 1)

    def both():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        run("c128", s1)
        run("c64", s2)
        e1, e2 = torch.cuda.Event(), torch.cuda.Event()
        e1.record(s1)
        e2.record(s2)
        torch.cuda.current_stream().wait_event(e1)
        torch.cuda.current_stream().wait_event(e2)

    def seq():
        run("c128", torch.cuda.current_stream())
        run("c64", torch.cuda.current_stream())

    res = {}
    for cap in ("", "148", "222"):
        if cap:
            os.environ["XFT_GRID_CAP"] = cap
        else:
            os.environ.pop("XFT_GRID_CAP", None)
        res[f"cap{cap or 'none'}"] = {
            "c64": timed(lambda: run("c64", torch.cuda.current_stream())),
            "c128": timed(lambda: run("c128", torch.cuda.current_stream())),
            "seq": timed(seq),
            "concurrent": timed(both),
        }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
