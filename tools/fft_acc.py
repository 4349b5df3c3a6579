"""FFT accuracy probe: GPU dft_rows (c128) vs numpy's FFT (pocketfft) on random rows; relative L2
per size and sign, plus the Mehler path on config-3 row 992 against numpy (prototype of the same
windowed convolution in float64).  python tools/fft_acc.py"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import use_variant  # noqa: E402

use_variant()
import torch  # noqa: E402

from paper_0912_1379_b200 import ops  # noqa: E402

rng = np.random.default_rng(0)
for M in (256, 1024, 4096, 8192, 16384, 32768):
    x = rng.normal(size=(8, M)) + 1j * rng.normal(size=(8, M))
    for sign in (-1, 1):
        got = ops.dft_rows(torch.from_numpy(x).cuda(), sign).cpu().numpy()
        ref = np.fft.fft(x, axis=1) if sign < 0 else np.fft.ifft(x, axis=1) * M
        e = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print(f"M {M:6d} sign {sign:+d} rel L2 max {e.max():.2e} mean {e.mean():.2e}", flush=True)
