"""Run the reference's OWN pure tests against this package (gate iii).

A throw-away shim package named ``mgwfbp`` re-exports ``paper_1811_11141_b200`` (and its
submodules), then pytest runs a temporary copy of /root/reference/pkg/tests with that shim
first on sys.path.  Only tests that need no GPU are selected; the by-design failing
criterion 3 is deselected (test_acceptance.py::test_criterion_3_same_counterexamples_as_reference
pins its exact outcome instead).  Skipped where /root/reference is absent (the GPU box).
"""

import os
import pathlib
import shutil
import subprocess
import sys

import pytest

REF_TESTS = pathlib.Path("/root/reference/pkg/tests")
ROOT = pathlib.Path(__file__).resolve().parents[1]

SHIM = '''
import importlib, sys
_pkg = importlib.import_module("paper_1811_11141_b200")
from paper_1811_11141_b200 import *  # noqa
from paper_1811_11141_b200 import __version__  # noqa
for _name in ("allreduce_net", "cli", "comm_model", "merge_planner", "model_profile", "schedule_sim"):
    sys.modules[__name__ + "." + _name] = importlib.import_module("paper_1811_11141_b200." + _name)
'''

DESELECT = [
    "test_acceptance.py::test_criterion_3_planner_vs_oracle",   # fails by design in the reference too
    "test_acceptance.py::test_criterion_7_collective_correctness",  # data path: needs GPUs
    "test_acceptance.py::test_criterion_8_calibrate_then_predict",  # data path: needs GPUs
    "test_allreduce_net.py::test_ring_allreduce_exact_and_counters",
    "test_allreduce_net.py::test_ring_allreduce_payload_smaller_than_ring",
    "test_allreduce_net.py::test_length_mismatch_is_a_protocol_error",
    "test_allreduce_net.py::test_multi_frame_rounds",
    "test_allreduce_net.py::test_bench_local_measurement_shape",
    "test_allreduce_net.py::test_emulate_local_verified_report",
    "test_cli.py::test_bench_writes_fittable_csv",
    "test_cli.py::test_emulate_smoke",
    "test_cli.py::test_worker_subcommand_pair",
]


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tests not mounted (GPU box)")
def test_reference_pure_suite_passes_against_this_package(tmp_path):
    shim = tmp_path / "shim" / "mgwfbp"
    shim.mkdir(parents=True)
    (shim / "__init__.py").write_text(SHIM)
    (shim / "__main__.py").write_text("from paper_1811_11141_b200.cli import main\nraise SystemExit(main())\n")
    tests = tmp_path / "tests"
    shutil.copytree(REF_TESTS, tests)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(shim.parent), str(ROOT)])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["CUDA_VISIBLE_DEVICES"] = ""
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", str(tests), "--rootdir", str(tmp_path)]
    for d in DESELECT:
        cmd += ["--deselect", "tests/" + d]
    proc = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join(proc.stdout.splitlines()[-25:])
    assert proc.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
