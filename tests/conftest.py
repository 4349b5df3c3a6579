import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")
    config.addinivalue_line("markers", "slow: long-running check")


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "golden.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def rel_l2(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (scale if scale else 1.0))


def max_row_rel_l2(got, ref):
    got = np.atleast_2d(np.asarray(got))
    ref = np.atleast_2d(np.asarray(ref))
    num = np.linalg.norm(got - ref, axis=-1)
    den = np.linalg.norm(ref, axis=-1)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(num / den))
