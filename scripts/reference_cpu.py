"""Time the UNMODIFIED reference (its own CLI, `python -m mgwfbp emulate`, loopback TCP ring,
Python compute agent) beside the oracle port that bench.py's reference arm runs, on the same
B200-class ResNet-50 profile and the WFBP plan (= the MG-WFBP plan at B200 speed).

Runs only where /root/reference exists (this container; it does not travel to the GPU box):

    python scripts/reference_cpu.py [--nodes 2,4,8] [--iterations 20] > profiles/reference_cpu_r01.json
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF_SRC = pathlib.Path("/root/reference/pkg/src")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", default="2,4,8")
    ap.add_argument("--iterations", type=int, default=20)
    args = ap.parse_args()
    if not REF_SRC.exists():
        raise SystemExit("the reference is not present here")
    import bench
    from oracle import emulation
    from paper_1811_11141_b200 import MergePlan, save_plan, save_profile

    profile, bwd, fwd = bench.b200_profile()
    plan = MergePlan(frozenset(), profile.num_layers)
    out = {"workload": "resnet50_like, B200-class timings (bench.b200_profile), WFBP plan (54 groups)",
           "host_cores": os.cpu_count(), "iterations": args.iterations, "rows": []}
    with tempfile.TemporaryDirectory() as tmp:
        prof_path, plan_path = pathlib.Path(tmp, "profile.json"), pathlib.Path(tmp, "plan.json")
        save_profile(profile, prof_path)
        save_plan(plan, plan_path)
        for n in [int(x) for x in args.nodes.split(",")]:
            rep = pathlib.Path(tmp, f"ref_{n}.json")
            env = dict(os.environ, PYTHONPATH=str(REF_SRC))
            cmd = [sys.executable, "-m", "mgwfbp", "emulate", "--profile", str(prof_path), "--nodes", str(n),
                   "--plan", str(plan_path), "--iterations", str(args.iterations), "--warmup", "2", "--out", str(rep)]
            subprocess.run(cmd, env=env, check=True, capture_output=True, text=True, timeout=1800)
            reports = json.loads(rep.read_text())
            ref_ms = max(r["mean_seconds"] for r in (reports if isinstance(reports, list) else reports.values())) * 1e3
            walls, ok = emulation.emulate(profile, plan, n, args.iterations, warmup=2)
            out["rows"].append({"nodes": n, "reference_ms": round(ref_ms, 3),
                                "oracle_port_ms": round(statistics.fmean(walls) * 1e3, 3), "port_verified": ok})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
