"""ncu workload: exactly the bench's N=1 MG-WFBP iteration (B200 ResNet-50 profile, the
plan bench.py derives, CUDA graph, per-group fill + one fused group kernel), run ITERS times.

    ncu --set full --kernel-name-base demangled -k regex:'fused_oneshot_kernel<1>' \\
        python scripts/profile_step.py --iters 1

writes the per-group algorithmic bytes of the fused N=1 kernel (4 x group bytes: read
layers, write bucket, read bucket, write layers) as JSON so scripts/summarize_step.py can
pair them with ncu's per-launch dram bytes.
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/profile_step_groups.json")
    args = ap.parse_args()
    import torch

    from paper_1811_11141_b200 import find_merge_plan
    from paper_1811_11141_b200.overlap import OverlappedIteration

    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    profile, _, _ = bench.b200_profile()
    exch = bench._exchange_times(None, 1, device, bench.FIT_SIZES, kind=0, repeats=3, warmups=1)
    model, _ = bench._fit(bench.FIT_SIZES, exch, 1)
    plan = find_merge_plan(profile, model)
    it = OverlappedIteration(profile, plan, comm=None, rank=0, world=1, device=device, graph=True, fused=True)
    try:
        for _ in range(args.iters):
            it.run()
        torch.cuda.synchronize()
        ok = it.verify()
        groups = [b for b in it.group_bytes() if b]
    finally:
        it.close()
    out = {"groups": len(groups), "algorithmic_bytes": [4 * b for b in groups], "verified": bool(ok),
           "kernel": "fused K1+K4 (N=1)"}
    pathlib.Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    pathlib.Path(args.out).write_text(json.dumps(out))
    print(json.dumps({k: out[k] for k in ("groups", "verified")}))


if __name__ == "__main__":
    main()
