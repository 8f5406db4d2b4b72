"""The CLI data verbs on GPUs (the reference's test_cli.py:163-204 for bench / emulate /
worker, here over NVLink): `bench` writes the measurement CSV, `emulate` reports verified
iterations, a hand-launched `worker` pair meets and measures, and a worker whose peer never
comes exits 2 (ring failure) -- that one, and `bench --local-group`, need a single GPU only."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_devices
from paper_1811_11141_b200 import load_measurements, resnet50_like, save_profile
from paper_1811_11141_b200.allreduce_net import _free_port

pytestmark = pytest.mark.gpu

CLI = [sys.executable, "-m", "paper_1811_11141_b200"]


def _run(args, timeout=240):
    return subprocess.run(CLI + args, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.fixture
def two_gpus():
    if cuda_devices() < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU)")


def test_bench_verb_writes_csv(tmp_path, two_gpus):
    out = tmp_path / "bench.csv"
    proc = _run(["bench", "--nodes", "2", "--sizes", "4096,65536,1048576", "--repeats", "2", "--warmups", "1",
                 "--out", str(out)])
    assert proc.returncode == 0, proc.stderr
    ms = load_measurements(out)
    assert [m.nbytes for m in ms] == [4096, 65536, 1048576]
    assert all(m.n_nodes == 2 and 0 < m.seconds < 1e-2 for m in ms)


def test_bench_verb_local_group_on_one_gpu(tmp_path):
    """`bench --local-group`: the reference's bench verb through the real protocol with every
    rank's CTAs in one cooperative launch on a single GPU (exact sums checked inside)."""
    out = tmp_path / "bench.csv"
    proc = _run(["bench", "--nodes", "4", "--local-group", "--sizes", "4096,65536,1048576,4194304", "--repeats", "2",
                 "--warmups", "1", "--out", str(out)])
    assert proc.returncode == 0, proc.stderr
    ms = load_measurements(out)
    assert [m.nbytes for m in ms] == [4096, 65536, 1048576, 4194304]
    assert all(m.n_nodes == 4 and 0 < m.seconds < 1e-2 for m in ms)
    assert "fitted: a=" in proc.stdout


def test_emulate_verb_verified(tmp_path, two_gpus):
    ppath = tmp_path / "profile.json"
    save_profile(resnet50_like(backward_seconds=2e-3, forward_seconds=1e-3), ppath)
    plan = tmp_path / "plan.json"
    plan.write_text("[2, 3, 4]\n")
    report = tmp_path / "report.json"
    events = tmp_path / "events.csv"
    proc = _run(["emulate", "--profile", str(ppath), "--nodes", "2", "--plan", str(plan), "--iterations", "3",
                 "--warmup", "1", "--out", str(report), "--events-csv", str(events)])
    assert proc.returncode == 0, proc.stderr
    assert "verified=True" in proc.stdout
    doc = json.loads(report.read_text())
    assert set(doc) == {"0", "1"} and all(d["verified"] for d in doc.values())
    rows = events.read_text().splitlines()
    assert rows[0] == "layer,kind,start_s,end_s"
    kinds = [r.split(",")[1] for r in rows[1:]]
    assert kinds.count("backward") == 54 and kinds.count("comm") == 51  # groups {2,3,4} -> 51 messages


def test_worker_subcommand_pair(tmp_path, two_gpus):
    port = _free_port("127.0.0.1")
    base = CLI + ["worker", "--role", "bench", "--nodes", "2", "--base-port", str(port), "--sizes", "4096,16384",
                  "--repeats", "1", "--warmups", "0"]
    out_csv = tmp_path / "bench.csv"
    p0 = subprocess.Popen(base + ["--rank", "0", "--out", str(out_csv)], stdout=subprocess.PIPE, text=True, cwd=ROOT)
    p1 = subprocess.Popen(base + ["--rank", "1"], stdout=subprocess.PIPE, text=True, cwd=ROOT)
    assert p0.wait(timeout=180) == 0
    assert p1.wait(timeout=180) == 0
    assert [m.nbytes for m in load_measurements(out_csv)] == [4096, 16384]


def test_worker_network_failure_exits_two():
    """Nobody else joins: the rendezvous times out -> exit 2 (ring failure), on one GPU."""
    if cuda_devices() < 1:
        pytest.skip("needs a CUDA device")
    port = _free_port("127.0.0.1")
    proc = _run(["worker", "--role", "bench", "--rank", "0", "--nodes", "2", "--base-port", str(port),
                 "--device", "0", "--timeout", "1.5"], timeout=120)
    assert proc.returncode == 2, (proc.returncode, proc.stderr[-500:])
    assert "could not join" in proc.stderr
