"""Config-3 row 992 (worst row of the all-rows check) through the GPU alone, in a small batch, and in
the full batch, against a float64 numpy FFT convolution of the same windowed factorisation
(tools/ for the accuracy investigation).  python tools/mehler_row_probe.py"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

print("library:", use_variant())
import torch  # noqa: E402

from paper_0912_1379_b200 import dense, mehler, workloads  # noqa: E402

c3 = workloads.config3()
z = c3.extra["z"]
n = 16384
r = 992
f = c3.values[r]
zz = complex(z[r])
half = math.pi / math.sqrt(2 * n) / 2
x = (2 * np.arange(n) - n + 1) * half
one = 1 - zz * zz
A = np.sqrt(2 / one)
Q = 2 * zz / one
sigma = 1 if Q.real >= 0 else -1
gam = (1 - zz) / (2 * (1 + zz)) if sigma > 0 else (1 + zz) / (2 * (1 - zz))
kk = math.ceil(math.sqrt(46 / gam.real) / (2 * half)) + 1
k0 = n // 2 - kk
wn = n - 2 * k0
k = k0 + np.arange(wn)
ks = k if sigma > 0 else n - 1 - k
u = np.exp(-gam * x[k] ** 2) * f[ks]
beta = 2 * sigma * Q * half * half
l = np.arange(-(wn - 1), wn).astype(float)
h = np.exp(-beta * l ** 2)
M = 1
while M < 2 * wn - 1:
    M *= 2
hp = np.zeros(M, complex)
hp[:wn] = h[wn - 1:]
hp[M - (wn - 1):] = h[:wn - 1]
up = np.zeros(M, complex)
up[:wn] = u
c = np.fft.ifft(np.fft.fft(up) * np.fft.fft(hp))[:wn]
ref = np.zeros(n, complex)
ref[k0:k0 + wn] = A * 2 * half * np.exp(-gam * x[k] ** 2) * c


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


alone = mehler.mehler_rows(torch.from_numpy(f[None, :].copy()).cuda(), [zz]).cpu().numpy()[0]
small = mehler.mehler_rows(torch.from_numpy(c3.values[r - 2:r + 2].copy()).cuda(), z[r - 2:r + 2]).cpu().numpy()[2]
full = mehler.mehler_rows(torch.from_numpy(c3.values).cuda(), z).cpu().numpy()[r]
dn = dense.dense_mehler_apply(torch.from_numpy(f[None, :].copy()).cuda(), [zz]).cpu().numpy()[0]
print("M", M, "wn", wn, "k0", k0)
print("alone vs numpy-fft", rel(alone, ref), " small-batch", rel(small, ref), " full-batch", rel(full, ref))
print("gpu dense vs numpy-fft", rel(dn, ref))
# which factor: test with f = unit impulse at the window centre and a smooth Gaussian
for name, g in (("impulse", np.eye(1, n, n // 2)[0].astype(complex)), ("gauss", np.exp(-x * x / 2).astype(complex))):
    got = mehler.mehler_rows(torch.from_numpy(g[None, :].copy()).cuda(), [zz]).cpu().numpy()[0]
    uu = np.exp(-gam * x[k] ** 2) * g[ks]
    up2 = np.zeros(M, complex)
    up2[:wn] = uu
    c2 = np.fft.ifft(np.fft.fft(up2) * np.fft.fft(hp))[:wn]
    ref2 = np.zeros(n, complex)
    ref2[k0:k0 + wn] = A * 2 * half * np.exp(-gam * x[k] ** 2) * c2
    print(name, "gpu vs numpy", rel(got, ref2))
