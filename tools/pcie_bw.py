"""Pinned host <-> device copy bandwidth (one direction, and both at once on two streams)."""
import json
import torch

n = 400 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


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


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = t(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_b, non_blocking=True))
bo = t(both)
print(json.dumps({"h2d_GBps": n / h2d / 1e6, "d2h_GBps": n / d2h / 1e6, "duplex_GBps_each": n / bo / 1e6}))
