"""Tuning-only: point the package at a variant build (tools/build_variant.sh) named by $XFT_LIB.

The product loader (_native.py) only ever loads the in-tree libxft_b200.so; A/B
scripts call use_variant() before the first transform instead.
"""
import os


def use_variant():
    path = os.environ.get("XFT_LIB")
    if path:
        from paper_0912_1379_b200 import _native

        _native._lib = _native.load_library(path)
    return path or "default"
