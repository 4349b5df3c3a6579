import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_0912_1379_b200 import mehler, workloads
g = np.load('/root/repo/tests/golden/mehler_truth_cfg3.npz')
c3 = workloads.config3(); rows = [int(r) for r in g['rows']]; js = g['js']
got = mehler.mehler_rows(torch.from_numpy(c3.values[rows]).cuda(), c3.extra['z'][rows]).cpu().numpy()
for i, r in enumerate(rows):
    t = g[f'truth_{r}']; print(r, np.linalg.norm(got[i, js] - t) / np.linalg.norm(t))
