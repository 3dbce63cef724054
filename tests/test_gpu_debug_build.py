"""The parity suite under the debug build (libgs_debug.so: every index a
kernel derives from another kernel's output is bounds-checked on the device,
gs_internal.cuh GS_ASSERT; a failed check traps and fails the launch).
compute-sanitizer is closed on this pool; this is its substitute."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suite_under_bounds_checks():
    lib = os.path.join(ROOT, "paper_2312_10070_b200", "libgs_debug.so")
    assert os.path.exists(lib), "build the debug library: GS_DEBUG=1 python -m paper_2312_10070_b200._build"
    assert b"GS_ASSERT failed" in open(lib, "rb").read()  # the checks are compiled in
    tests = ["tests/test_gpu_parity.py", "tests/test_gpu_fused_l1.py", "tests/test_gpu_pipeline.py",
             "tests/test_gpu_fullsize.py"]
    p = subprocess.run([sys.executable, "-m", "pytest", "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider"] + tests,
                       cwd=ROOT, env=dict(os.environ, GS_LIB_DEBUG="1"), capture_output=True, text=True,
                       timeout=1800)
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-2000:])
    assert "GS_ASSERT failed" not in p.stdout + p.stderr
