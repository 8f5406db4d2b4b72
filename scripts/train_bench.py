"""Real training step (torchvision ResNet-50, bs 32/GPU, fp32, SGD): MG-WFBP vs WFBP vs
SyncEASGD on the B200 kernels, vs PyTorch DDP (NCCL), vs compute only.  torchrun, one
rank per GPU; prints one JSON document on rank 0.

    torchrun --nproc-per-node N scripts/train_bench.py [--steps 20] [--model resnet50]

Gradient readiness comes from autograd (paper_1811_11141_b200.autograd); the merge plan
comes from a per-parameter backward profile measured here and the (a, b) fitted on this
box, exactly the reference's calibrate -> plan -> run workflow.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--ctas", default="296,64,32,16", help="CTA caps to try for the overlapped collectives")
    ap.add_argument("--priorities", default="0,-1", help="comm stream priorities to try")
    ap.add_argument("--gates", default="0,1", help="peer gate off/on variants to try")
    ap.add_argument("--bf16", action="store_true",
                    help="bf16 parameters and gradients (bf16 wire, fp32 accumulation in the exchange)")
    ap.add_argument("--tune", action="store_true",
                    help="interference-aware MG-WFBP: pick the startup scale k by measured step time "
                         "(replan.calibrate_startup) at each CTA cap, then time the chosen plan")
    ap.add_argument("--a-scales", default="", help="extra MG-WFBP plans under an inflated startup a (e.g. 4,16): "
                    "probes whether merging more pays once interference with backward is priced in")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import torchvision

    from paper_1811_11141_b200 import MergePlan, find_merge_plan, simulate_mgwfbp, simulate_sync_easgd, simulate_wfbp
    from paper_1811_11141_b200.allreduce_net import open_session_dist
    from paper_1811_11141_b200.autograd import MergedGradientSync, measure_profile, trainable_parameters

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    torch.manual_seed(0)
    dtype = torch.bfloat16 if args.bf16 else torch.float32
    net = getattr(torchvision.models, args.model)().to(device=device, dtype=dtype)
    params = trainable_parameters(net)
    total = sum(p.numel() for p in params)
    gen = torch.Generator(device=device).manual_seed(1000 + rank)
    x = torch.randn(args.batch, 3, 224, 224, device=device, generator=gen).to(dtype)
    y = torch.randint(0, 1000, (args.batch,), device=device, generator=gen)
    loss_fn = torch.nn.CrossEntropyLoss()

    def step():
        return loss_fn(net(x), y)

    # 1. calibrate: per-parameter backward profile (rank 0's, shared) and (a, b) on this box
    prof = measure_profile(net, step, name=f"{args.model}-bs{args.batch}-measured")
    if world > 1:
        box = [prof]
        dist.broadcast_object_list(box, src=0)
        prof = box[0]
    session = comm = None
    if world > 1:
        _, session = open_session_dist(capacity_bytes=4 * total)  # fp32-sized: also holds bf16 buckets
        comm = session.comm
    # (a, b) of the exchange the run will use: bf16 group exchange (kind 5) for bf16 gradients
    exch = bench._exchange_times(comm, world, device, bench.FIT_SIZES,
                                 kind=(5 if args.bf16 else 4) if world > 1 else 0)
    model_ab, _ = bench._fit(bench.FIT_SIZES, exch, world)
    n = prof.num_layers
    plans = {"wfbp": MergePlan(frozenset(), n), "mgwfbp": find_merge_plan(prof, model_ab),
             "synceasgd": MergePlan(frozenset(range(2, n + 1)), n)}
    predicted = {"wfbp": simulate_wfbp(prof, model_ab), "mgwfbp": simulate_mgwfbp(prof, model_ab, plans["mgwfbp"]),
                 "synceasgd": simulate_sync_easgd(prof, model_ab)}
    from paper_1811_11141_b200 import CommModel

    for k in [float(x) for x in args.a_scales.split(",") if x]:
        inflated = CommModel(model_ab.a * k, model_ab.b)
        name = f"mgwfbp_a{k:g}x"
        plans[name] = find_merge_plan(prof, inflated)
        predicted[name] = simulate_mgwfbp(prof, inflated, plans[name])

    def timed(run_one, label):
        s = torch.cuda.current_stream()
        for _ in range(args.warmup):
            run_one()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            run_one()
            b.record(s)
            ts.append((a, b))
        torch.cuda.synchronize()
        vals = [u.elapsed_time(v) for u, v in ts]
        vals = bench._max_over_ranks(vals, world, device)
        return {"ms_mean": round(statistics.fmean(vals), 4), "ms_median": round(statistics.median(vals), 4)}

    opt = torch.optim.SGD(net.parameters(), lr=1e-3, momentum=0.9)
    results = {}

    def local_step():
        opt.zero_grad(set_to_none=False)
        step().backward()
        opt.step()

    results["compute_only"] = timed(local_step, "compute_only")
    variants = [(int(c), int(p), int(g)) for c in args.ctas.split(",") for p in args.priorities.split(",")
                for g in args.gates.split(",")]
    for cap, prio, gate in variants:
        for name in plans:
            sync = MergedGradientSync(params, plans[name], comm=comm, world=world, scale=1.0 / world,
                                      sync_after_backward=name == "synceasgd", max_ctas=cap, priority=prio,
                                      gate=bool(gate))

            def synced_step():
                opt.zero_grad(set_to_none=False)
                step().backward()
                sync.finish()
                opt.step()

            key = f"{name}_ctas{cap}" + ("_hiprio" if prio < 0 else "") + ("_gate" if gate else "")
            results[key] = timed(synced_step, key)
            results[key].update({"groups": len(plans[name].groups()),
                                 "launched_per_step": sync.launched // (args.warmup + args.steps),
                                 "predicted_t_iter_ms": round(predicted[name].t_iter * 1e3, 4),
                                 "predicted_t_c_no_us": round(predicted[name].t_c_no * 1e6, 2)})
            # consistency: every rank holds bit-identical reduced gradients
            if world > 1:
                flat = torch.cat([p.grad.reshape(-1) for p in params])
                lo, hi = flat.clone(), flat.clone()
                dist.all_reduce(lo, op=dist.ReduceOp.MIN)
                dist.all_reduce(hi, op=dist.ReduceOp.MAX)
                results[key]["ranks_bit_identical"] = bool(torch.equal(lo, hi))
            sync.close()
        if world == 1:
            break
    if args.tune and world > 1:
        from paper_1811_11141_b200.replan import calibrate_startup

        for cap in [int(c) for c in args.ctas.split(",")]:
            def synced(plan, steps, warm):
                sync = MergedGradientSync(params, plan, comm=comm, world=world, scale=1.0 / world, max_ctas=cap,
                                          priority=-1)

                def synced_step():
                    opt.zero_grad(set_to_none=False)
                    step().backward()
                    sync.finish()
                    opt.step()

                saved = args.steps, args.warmup
                args.steps, args.warmup = steps, warm
                try:
                    res = timed(synced_step, "tune")
                finally:
                    args.steps, args.warmup = saved
                    sync.close()
                return res

            # timed() already takes the max over ranks, so every rank sees the same numbers
            k, plan, times = calibrate_startup(prof, model_ab, lambda p: synced(p, 10, 3)["ms_mean"],
                                               scales=(1, 2, 4, 8, 16, 32, 64))
            key = f"mgwfbp_tuned_ctas{cap}_hiprio"
            results[key] = synced(plan, args.steps, args.warmup)
            results[key].update({"groups": len(plan.groups()), "startup_scale": k,
                                 "calibration_ms": {str(kk): round(v, 4) for kk, v in times.items()}})
    if world > 1:
        ddp = torch.nn.parallel.DistributedDataParallel(net, device_ids=[local], gradient_as_bucket_view=True,
                                                      broadcast_buffers=False)
        opt2 = torch.optim.SGD(ddp.parameters(), lr=1e-3, momentum=0.9)

        def ddp_step():
            opt2.zero_grad(set_to_none=False)
            loss_fn(ddp(x), y).backward()
            opt2.step()

        results["ddp_nccl"] = timed(ddp_step, "ddp")
    if session is not None:
        session.raise_if_failed()
        session.close()
    out = {
        "workload": f"torchvision {args.model}, batch {args.batch} per GPU, {'bf16' if args.bf16 else 'fp32'}, "
                    f"SGD momentum, synthetic data",
        "world": world, "params": total, "layers": n,
        "measured_forward_ms": round(prof.forward_time * 1e3, 3),
        "measured_backward_ms": round(prof.total_backward_time * 1e3, 3),
        "fitted_a_us": round(model_ab.a * 1e6, 3), "fitted_b_ns_per_byte": model_ab.b * 1e9,
        "mgwfbp_groups": len(plans["mgwfbp"].groups()),
        "results": results,
    }
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
