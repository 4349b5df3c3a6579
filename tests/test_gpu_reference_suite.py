"""The reference's own test suite (pkg/tests, 259 tests) run against the GPU package.

``oracle/build_ref.sh`` ships the reference's test files as
``oracle/_ref/reference_tests``; ``tests/ref_shim/xft`` serves the ``xft``
namespace those files import: every hot-path name from
``paper_0912_1379_b200`` (GPU), the out-of-scope helpers (exact Hermite zeros,
eigen-FrFT, quadrature/closed-form oracles, calibration constants) from the
reference itself.  The suite runs in a subprocess; every failure must be one of
the documented EXPECTED_FAILURES (with the reason), and no more.
The per-test outcome table is written to gpurun_out/reference_suite.xml when
that directory exists (evidence for DESIGN.md).
"""
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "reference_tests")

pytestmark = pytest.mark.gpu

# test id suffix -> why it cannot pass against this build (fails by design)
EXPECTED_FAILURES = {
    # criterion 4 fails in the reference itself (pkg/test_output.txt records 258/259)
    "test_04_convergence_order_fourier": "fails by design in the reference too",
    # `grid --exact` (exact Hermite zeros) is outside this build: exit 2
    "TestGrid::test_exact_grid": "grid --exact is out of scope",
    # the brute-force quadrature oracle is outside this build: exit 2
    "TestCompare::test_quadrature_oracle": "--oracle quadrature is out of scope",
}


def _expected(test_id):
    return next((why for k, why in EXPECTED_FAILURES.items() if k in test_id), None)


def test_reference_suite_against_gpu_package(tmp_path):
    if not os.path.isdir(SUITE):
        pytest.skip("oracle/_ref/reference_tests missing (run oracle/build_ref.sh where /root/reference exists)")
    xml = tmp_path / "suite.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "ref_shim"), ROOT])
    proc = subprocess.run([sys.executable, "-m", "pytest", SUITE, "-q", "-p", "no:cacheprovider", "-rf",
                           f"--junitxml={xml}", "--rootdir", SUITE],
                          cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1800)
    out_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, "reference_suite.log"), "w") as f:
            f.write(proc.stdout[-20000:] + "\n" + proc.stderr[-5000:])
        if xml.exists():
            with open(os.path.join(out_dir, "reference_suite.xml"), "w") as f:
                f.write(xml.read_text())
    assert xml.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    root = ET.parse(xml).getroot()
    total, failed = 0, []
    for case in root.iter("testcase"):
        total += 1
        tid = f"{case.get('classname', '')}::{case.get('name')}"
        if case.find("failure") is not None or case.find("error") is not None:
            failed.append(tid)
    unexpected = [t for t in failed if _expected(t) is None]
    assert total >= 250, f"only {total} reference tests collected\n{proc.stdout[-3000:]}"
    assert not unexpected, "unexpected failures:\n" + "\n".join(unexpected) + "\n" + proc.stdout[-6000:]
