"""Launch one BASELINE config's transform a few times (for ncu launch lists / captures).

  python tools/prof_cfg.py cfg5|cfg3|cfg2|cfg4 [reps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    cfg = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    import torch

    from paper_0912_1379_b200 import lct2d, mehler, ops, workloads

    if cfg == "cfg5":
        f = torch.from_numpy(workloads.config5_field(16384)).cuda()
        out, ws = torch.empty_like(f), torch.empty_like(f)
        for _ in range(reps):
            lct2d.lct2d(f, workloads.CONFIG5_ABCD, workloads.CONFIG5_ABCD, out=out, workspace=ws)
    elif cfg == "cfg3":
        c = workloads.config3()
        v = torch.from_numpy(c.values).cuda()
        o = torch.empty_like(v)
        for _ in range(reps):
            mehler.mehler_rows(v, c.extra["z"], out=o)
    elif cfg in ("cfg2", "cfg2c64", "cfg2c128"):
        dts = {"cfg2": (np.complex64, np.complex128), "cfg2c64": (np.complex64,), "cfg2c128": (np.complex128,)}[cfg]
        for dt in dts:
            c = workloads.config2(dtype=dt)
            v = torch.from_numpy(c.values).cuda()
            p = torch.from_numpy(c.abcd).cuda()
            o = torch.empty_like(v)
            for _ in range(reps):
                ops.lct_rows(v, p, out=o, validate=False)
    elif cfg == "cfg4":
        c = workloads.config4()
        v = torch.from_numpy(c.values).cuda()
        o = torch.empty_like(v)
        for _ in range(reps):
            ops.lct_rows(v, c.abcd, out=o, validate=False)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
