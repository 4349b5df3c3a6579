"""Config-3: every row's fast-vs-dense-GPU relative L2 error, the worst rows listed with their z, m,
window class and the error's location; the worst rows' GPU outputs saved for host long-double checks.
python tools/mehler_allrows.py [outdir]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

print("library:", use_variant())
import torch  # noqa: E402

from paper_0912_1379_b200 import dense, mehler, workloads  # noqa: E402

out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
c3 = workloads.config3()
z, m = c3.extra["z"], c3.extra["m"]
v = torch.from_numpy(c3.values).cuda()
got = mehler.mehler_rows(v, z).cpu().numpy()
errs, ref_all = [], np.empty_like(got)
for s in range(0, z.shape[0], 128):
    ref_all[s:s + 128] = dense.dense_mehler_apply(v[s:s + 128], z[s:s + 128]).cpu().numpy()
e = np.linalg.norm(got - ref_all, axis=1) / np.linalg.norm(ref_all, axis=1)
gam = np.where((2 * z / (1 - z * z)).real >= 0, (1 - z) / (2 * (1 + z)), (1 + z) / (2 * (1 - z))).real
order = np.argsort(e)[::-1]
print("rows with rel err > 1e-12:", int((e > 1e-12).sum()), " > 1e-13:", int((e > 1e-13).sum()))
for r in order[:25]:
    d = np.abs(got[r] - ref_all[r])
    j = int(np.argmax(d))
    print(f"row {r:4d} err {e[r]:.2e} z {z[r]:.4f} |z| {abs(z[r]):.3f} m {m[r]:2d} gam {gam[r]:.3e} "
          f"|1-z2| {abs(1 - z[r] ** 2):.3f} argmax {j} |g|max {np.abs(ref_all[r]).max():.2e}")
np.savez_compressed(os.path.join(out_dir, "mehler_worst.npz"), rows=order[:25], got=got[order[:25]],
                    dense=ref_all[order[:25]], err=e)
