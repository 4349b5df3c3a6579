"""Launch each hot kernel a few times on a BASELINE-sized batch (for ncu captures).

  python tools/prof_kernels.py [--config cfg2] [--reps 3]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtypes", default="c64,c128")
    a = ap.parse_args()
    import torch

    from paper_0912_1379_b200 import ops, workloads

    if a.config == "cfg2":
        for tag in a.dtypes.split(","):
            dt = np.complex64 if tag == "c64" else np.complex128
            c = workloads.config2(dtype=dt)
            v = torch.from_numpy(c.values).cuda()
            p = torch.from_numpy(c.abcd).cuda()
            out = torch.empty_like(v)
            for _ in range(a.reps):
                ops.lct_rows(v, p, out=out, validate=False)
    elif a.config == "cfg4":
        c = workloads.config4()
        v = torch.from_numpy(c.values).cuda()
        out = torch.empty_like(v)
        for _ in range(a.reps):
            ops.lct_rows(v, c.abcd, out=out, validate=False)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
