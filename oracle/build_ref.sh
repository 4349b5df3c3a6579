#!/usr/bin/env bash
# Installs the reference package (/root/reference/pkg, pure Python + NumPy) into
# oracle/_ref/ -- TEST/BENCH INFRASTRUCTURE ONLY.
#
# oracle/_ref/ is git-ignored (never committed) but not gpurun-ignored, so the
# installed reference (and a copy of its test suite, reference_tests/) travels
# to the GPU box, where bench.py's CPU arms
# (`--impl reference`, `cpu_baseline`) import it to time the reference's own
# per-row fast_lct / fast_frft / mehler_kernel.  The product package never
# imports it.  The reference has no native code, so "building" it is a plain
# wheel install of its sources from a scratch copy (/root/reference is
# read-only and setuptools writes build metadata next to the sources).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${XFT_REFERENCE_PKG:-/root/reference/pkg}"
DEST="$HERE/_ref"
if [ ! -f "$SRC/pyproject.toml" ]; then
    echo "build_ref: $SRC not present; keeping the existing $DEST (if any)" >&2
    exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DEST"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$DEST" "$TMP/pkg"
# the reference's own test suite, run against the GPU package through tests/ref_shim
# (tests/test_gpu_reference_suite.py); like the package, never committed
cp -r "$SRC/tests" "$DEST/reference_tests"
python - "$DEST" <<'EOF'
import sys
sys.path.insert(0, sys.argv[1])
import xft
print(f"build_ref: xft {xft.__version__} installed into {sys.argv[1]}")
EOF
