"""BASELINE configs beyond the headline: every profile through WFBP / SyncEASGD /
MG-WFBP on the same kernels at N GPUs (torchrun), next to the simulator's predictions
under the (a, b) fitted on this box.

    torchrun --nproc-per-node N scripts/run_profiles.py [--steps 10]

Profiles (B200-class timings from profiles/backward_times_b200.json):
  googlenet_like(aux=False)  ~7M params, bs 64       (BASELINE config 0)
  resnet50_like              25.5M, bs 32            (config 1, the headline)
  vgg16_like                 138M, fc6 = 411 MB      (config 2, two-shot regime)
  bert_base_like             199 tensors, bs 32x128  (config 3, startup-dominated)
  synth_profile(1000, 4 KiB..64 MiB tensors)         (config 4), reference time scale
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def profiles():
    from paper_1811_11141_b200 import bert_base_like, googlenet_like, resnet50_like, synth_profile, vgg16_like

    doc = json.loads((bench.ROOT / "profiles" / "backward_times_b200.json").read_text())
    g, r, v, b = doc["googlenet_bs64"], doc["resnet50_bs32"], doc["vgg16_bs32"], doc["bert_base_bs32_seq128"]
    return [
        ("googlenet_noaux_bs64", googlenet_like(g["backward_s"], g["forward_s"], aux=False)),
        ("resnet50_bs32", resnet50_like(r["backward_s"], r["forward_s"])),
        ("vgg16_bs32", vgg16_like(v["backward_s"], v["forward_s"])),
        ("bert_base_bs32", bert_base_like(b["backward_s"], b["forward_s"])),
        ("synth_1000", synth_profile(1000, param_range=(1024, 16_777_216), seed=0)),
    ]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1811_11141_b200 import (
        MergePlan,
        find_merge_plan,
        simulate_mgwfbp,
        simulate_sync_easgd,
        simulate_wfbp,
    )
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    chosen = [(k, p) for k, p in profiles() if not args.only or k in args.only.split(",")]
    cap = max(4 * p.total_params for _, p in chosen)
    session = comm = None
    if world > 1:
        _, session = open_session_dist(capacity_bytes=cap)
        comm = session.comm
    exch = bench._exchange_times(comm, world, device, bench.FIT_SIZES, kind=4 if world > 1 else 0)
    model, fit_ok = bench._fit(bench.FIT_SIZES, exch, world)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device=device)
    ctx = bench.RankContext(rank, world, local, device, comm, session, flush)
    out = {"world": world, "fitted_a_us": model.a * 1e6, "fitted_b_ns_per_byte": model.b * 1e9, "profiles": {}}
    for key, prof in chosen:
        n = prof.num_layers
        plans = {"wfbp": MergePlan(frozenset(), n), "synceasgd": MergePlan(frozenset(range(2, n + 1)), n),
                 "mgwfbp": find_merge_plan(prof, model)}
        pred = {"wfbp": simulate_wfbp(prof, model), "synceasgd": simulate_sync_easgd(prof, model),
                "mgwfbp": simulate_mgwfbp(prof, model, plans["mgwfbp"])}
        entry = {"layers": n, "params": prof.total_params, "compute_s": prof.forward_time + prof.total_backward_time,
                 "mg_groups": len(plans["mgwfbp"].groups()), "strategies": {}}
        for name in ("wfbp", "synceasgd", "mgwfbp"):
            res, _, _, _, _ = bench.run_strategy(ctx, prof, plans[name], pred[name], args.steps, args.warmup)
            entry["strategies"][name] = res
        out["profiles"][key] = entry
        if rank == 0:
            print(key, json.dumps({k: (v["t_iter_ms"], v["t_c_no_us"], v["predicted_t_c_no_us"]) for k, v in entry["strategies"].items()}),
                  file=sys.stderr, flush=True)
    if session is not None:
        session.close()
    if rank == 0 and world > 1:
        # BASELINE config 0: the reference CPU path on the same GoogLeNet profile and N
        from oracle import emulation

        key, prof = profiles()[0]
        plan, cpu_model = bench._cpu_plan(prof, world)
        walls, ok = emulation.emulate(prof, plan, world, 10, warmup=1, time_budget_s=15.0)
        out["cpu_reference_" + key] = {"ranks": world, "t_iter_ms": sum(walls) / len(walls) * 1e3,
                                        "iterations": len(walls), "verified": ok, "plan_groups": len(plan.groups()),
                                        "fitted_a_us": None if cpu_model is None else cpu_model.a * 1e6}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
