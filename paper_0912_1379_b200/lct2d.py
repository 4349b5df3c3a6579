"""Separable 2-D LCT: fast LCT along axis 1 (rows), then along axis 0 (columns).

No reference symbol exists; the transform is defined as the composition of
the reference 1-D ``fast_lct`` (xft/lct.py:168-208) along both axes
(last row).  Single-GPU: ``xft_lct2d`` in libxft_b200.so.
"""
from __future__ import annotations

import numpy as np

from . import _native, ops
from .errors import ShapeError


def lct2d(field, abcd_row, abcd_col=None, *, out=None, workspace=None):
    """2-D LCT of a [n_rows, n_cols] complex CUDA tensor on one GPU."""
    torch = ops._torch()
    if abcd_col is None:
        abcd_col = abcd_row
    if field.dim() != 2 or not field.is_cuda:
        raise ShapeError("lct2d needs a 2-D CUDA tensor")
    f = field.contiguous()
    r, c = f.shape
    pr = np.ascontiguousarray(np.asarray(abcd_row, dtype=np.float64).reshape(4))
    pc = np.ascontiguousarray(np.asarray(abcd_col, dtype=np.float64).reshape(4))
    if out is None:
        out = torch.empty_like(f)
    if workspace is None:
        workspace = torch.empty_like(f)
    with torch.cuda.device(f.device):
        _native.call("xft_lct2d", f.data_ptr(), out.data_ptr(), r, c, ops._dtype_code(f),
                     pr.ctypes.data, pc.ctypes.data, workspace.data_ptr(), ops._stream_ptr(f.device))
    return out
