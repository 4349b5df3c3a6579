"""Graph-replayed timing of one batched row LCT (FrFT rows, alpha ~ U(0, pi)).

  python tools/time_rows.py --n 16384 --rows 16384 --dtype c64 [--reps 20]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

VARIANT = use_variant()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_0912_1379_b200 import ops

    rng = np.random.default_rng(5)
    al = rng.uniform(0, np.pi, a.rows)
    abcd = np.stack([np.cos(al), np.sin(al), -np.sin(al), np.cos(al)], 1)
    dt = np.complex64 if a.dtype == "c64" else np.complex128
    sets = []
    for _ in range(2):
        v = (rng.standard_normal((a.rows, a.n), dtype=np.float32) + 1j * rng.standard_normal((a.rows, a.n), dtype=np.float32)).astype(dt)
        tv = torch.from_numpy(v).cuda()
        sets.append((tv, torch.empty_like(tv), torch.from_numpy(abcd).cuda()))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for v, o, p in sets:
            ops.lct_rows(v, p, out=o, validate=False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(a.reps):
            v, o, p = sets[i % 2]
            ops.lct_rows(v, p, out=o, validate=False)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / a.reps)
    nbytes = sets[0][0].numel() * sets[0][0].element_size() * 2
    import hashlib

    sha = hashlib.sha256(sets[0][1].cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"variant": VARIANT, "sha": sha, "n": a.n, "rows": a.rows, "dtype": a.dtype, "us": round(best, 2),
                      "GBps": round(nbytes / best / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
