import sys, math, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle import xft_oracle as O
from paper_0912_1379_b200 import ops
rng = np.random.default_rng(3)
for n in [5000, 12000, 65536, 196608, 262144, 1048576]:
    for dt in (np.complex128, np.complex64):
        rows = 2
        al = np.array([0.7, 2.2])
        abcd = np.stack([np.cos(al), np.sin(al), -np.sin(al), np.cos(al)], 1)
        f = ((rng.standard_normal((rows, n)) + 1j*rng.standard_normal((rows, n)))/math.sqrt(2)).astype(dt)
        try:
            got = ops.lct_rows(torch.from_numpy(f).cuda(), abcd).cpu().numpy()
            _, ref = O.fast_lct_rows(abcd, f.astype(complex))
            err = np.max(np.linalg.norm(got-ref, axis=1)/np.linalg.norm(ref, axis=1))
            print(n, dt.__name__, 'rel_l2', err, flush=True)
        except Exception as e:
            print(n, dt.__name__, 'ERR', type(e).__name__, e, flush=True)
