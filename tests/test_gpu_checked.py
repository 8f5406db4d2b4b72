"""The bounds-checked build on the GPU (compute-sanitizer is closed on this pool): the
kernel and rank-group parity suites run once more in a subprocess against
libmgwfbp_b200_checked.so (-DMGW_CHECKED), where every tensor row walk, bucket / slot
index, barrier flag slot, LL area index and push row offset the kernels compute is
validated against its extent; the session must end with zero violations
(tests/conftest.py::_checked_build_violations) and the same bit-exact results."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_devices

pytestmark = pytest.mark.gpu

CHECKED = ROOT / "paper_1811_11141_b200" / "_lib" / "libmgwfbp_b200_checked.so"


def test_checked_build_zero_violations():
    if cuda_devices() < 1:
        pytest.skip("needs a CUDA device")
    if not CHECKED.exists():
        pytest.skip("checked library not built (python -c 'import __graft_entry__ as g; g.build()')")
    env = dict(os.environ, MGWFBP_B200_LIB=str(CHECKED))
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-m", "gpu", "-q", "-s", "-x", "-p", "no:cacheprovider",
         "tests/test_gpu_kernels.py", "tests/test_gpu_local_group.py", "tests/test_gpu_overlap.py"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = proc.stdout[-2000:] + proc.stderr[-1000:]
    assert proc.returncode == 0, tail
    assert "checked build: 0 index violations (checked=1)" in proc.stdout, tail
