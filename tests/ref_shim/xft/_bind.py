"""Loads the installed reference (oracle/_ref/xft) as ``xft_reference`` for the shim's
out-of-scope names, with its ``errors`` and ``lct`` modules bound to the GPU package's,
so reference helpers (oracle, calibration, exact eigen-FrFT) raise the same exception
classes and build the same parameter / signal types the GPU path consumes."""
import importlib.util
import os
import sys

import paper_0912_1379_b200.errors as _errors
import paper_0912_1379_b200.lct as _lct

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
REF = os.path.join(ROOT, "oracle", "_ref", "xft")


def reference():
    if "xft_reference" in sys.modules:
        return sys.modules["xft_reference"]
    if not os.path.isdir(REF):
        raise ImportError(f"{REF} missing: run oracle/build_ref.sh")
    sys.modules["xft_reference.errors"] = _errors
    sys.modules["xft_reference.lct"] = _lct
    spec = importlib.util.spec_from_file_location("xft_reference", os.path.join(REF, "__init__.py"),
                                                  submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["xft_reference"] = mod
    spec.loader.exec_module(mod)
    return mod
