"""MG-WFBP on B200: ResNet-50 iteration time at N GPUs (+ WFBP / SyncEASGD on the same
kernels, the fitted alpha/beta model, all-reduce bus GB/s vs size, rooflines).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1, one rank per GPU)

A *step* is one emulated training iteration (Algorithm 2) of the ResNet-50 layer
profile: simulated backward on a compute stream, every merge group packed (K1),
all-reduced over NVLink (K2/K3, N > 1) and unpacked (K4) on a comm stream as soon as
its head layer's gradient exists.  The headline is the MG-WFBP plan, planned from an
(a, b) fitted on this box; WFBP and SyncEASGD run on the same kernels.

Prints ONE JSON line on rank 0 (contract in the task statement).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ResNet-50 iter time + scaling eff. at 1/2/4/8 B200; allreduce bus GB/s vs size"
# Backward/forward seconds of torchvision ResNet-50 at the paper's batch size 32
# (PAPER.md:468), fp32 weights, measured on one B200 by scripts/measure_backward.py
# (profiles/backward_times_b200.json).  Only the totals enter resnet50_like(); the
# per-layer split is the reference's FLOPs proxy (model_profile.py:193-208).
PROFILE_TIMES = ROOT / "profiles" / "backward_times_b200.json"
FIT_SIZES = [1 << k for k in range(12, 27)]  # 4 KiB .. 64 MiB (BASELINE sweep)
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def b200_profile():
    from paper_1811_11141_b200 import resnet50_like

    bwd, fwd = 0.0171, 0.0085  # fallback if the measurement file is absent
    if PROFILE_TIMES.exists():
        doc = json.loads(PROFILE_TIMES.read_text())
        bwd, fwd = doc["resnet50_bs32"]["backward_s"], doc["resnet50_bs32"]["forward_s"]
    return resnet50_like(backward_seconds=bwd, forward_seconds=fwd), bwd, fwd


def peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        doc = json.loads(path.read_text())
        return float(doc["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


NVLINK_PEAK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal
L2_POLICY = ("GPU arm: a 256 MiB buffer (> 126 MB L2) is written and then read back between iterations, outside "
             "the timed events (the read-back evicts the dirty lines, so no write-back lands in the next iteration)")


def workload_config(bwd, fwd, world):
    """The workload keys both arms report identically (the driver compares them)."""
    return {
        "workload": "resnet50_like (54 layers, 25,503,912 fp32 params = 102,015,648 B), MG-WFBP iteration",
        "backward_s": bwd,
        "forward_s": fwd,
        "timings": "B200-class: torchvision ResNet-50 bs32 fwd/bwd measured on one B200, split by the "
                   "reference FLOPs proxy",
        "strategy": "mgwfbp",
        "parallelism": f"dp{world}",
        "l2": L2_POLICY,
    }


def l2_flush(buf):
    """Write then read a buffer larger than L2 on the current stream."""
    buf.zero_()
    buf.sum()


def host_cpu():
    """(cores this process may run on, CPU model) of the host."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = "unknown"
    try:
        for line in pathlib.Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


# --------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampling during the timed region (rank 0)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "250"],  # sparse: an NVML query can stall the GPU for ~1 ms
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        if self.proc is not None:
            time.sleep(1.0)  # NVML start-up stays out of the timed region
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if not getattr(self, "lines", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except (ValueError, IndexError):
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------- our arm


def _dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(values, world, device):
    import torch

    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def _exchange_times(comm, world, device, sizes, kind=0, algo=0, repeats=20, warmups=3):
    """Device seconds per exchange step (kind 0: pack + all-reduce + unpack, N=1: pack +
    unpack; kind 1: all-reduce kernel alone) per size: `repeats` back-to-back steps under
    one CUDA event pair (mgw_time_exchange), max over ranks."""
    import ctypes

    import torch

    from paper_1811_11141_b200 import _native

    stream = torch.cuda.Stream(device=device)
    out = []
    scratch = torch.ones(max(sizes) // 4, dtype=torch.float32, device=device)
    local_bucket = torch.empty_like(scratch) if world == 1 else None
    for nbytes in sizes:
        n = nbytes // (2 if (kind & 255) == 5 else 4)  # kind 5: bf16 elements
        table = _native.DeviceTable([(scratch.data_ptr(), n, 0)])
        sec = ctypes.c_double()
        _native.call("mgw_time_exchange", comm, table.ptr, 1, n,
                     None if local_bucket is None else local_bucket.data_ptr(), algo, kind,
                     repeats, warmups, ctypes.byref(sec), stream.cuda_stream)
        table.close()
        out.append(sec.value)
    return _max_over_ranks(out, world, device)


def _nccl_times(world, device, sizes, repeats=20, warmups=3, bf16=False):
    """ncclAllReduce (torch.distributed, comparison only), same loop timing."""
    import torch
    import torch.distributed as dist

    from paper_1811_11141_b200 import _native

    stream = torch.cuda.Stream(device=device)
    width = 2 if bf16 else 4
    buf = torch.ones(max(sizes) // width, dtype=torch.bfloat16 if bf16 else torch.float32, device=device)
    out = []
    with torch.cuda.stream(stream):
        for nbytes in sizes:
            x = buf[: nbytes // width]
            for _ in range(warmups):
                dist.all_reduce(x)
            _native.call("mgw_spin_ns", 1_000_000 + 20_000 * repeats, stream.cuda_stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(repeats):
                dist.all_reduce(x)
            b.record(stream)
            b.synchronize()
            out.append(a.elapsed_time(b) * 1e-3 / repeats)
    return _max_over_ranks(out, world, device)


def _allreduce_sweep(session, comm, world, device, sizes, with_nvls=False):
    """Bus GB/s vs size: our one-shot and two-shot kernels alone, the full group
    exchange (pack + all-reduce + unpack), and ncclAllReduce; the bf16 group exchange
    (bf16 wire, fp32 accumulation) vs NCCL bf16 at the same payload bytes."""
    from paper_1811_11141_b200 import _native

    one = _exchange_times(comm, world, device, sizes, kind=1, algo=_native.ALGO_ONESHOT)
    two = _exchange_times(comm, world, device, sizes, kind=1, algo=_native.ALGO_TWOSHOT)
    nccl = _nccl_times(world, device, sizes)
    session.raise_if_failed()
    nvls = None
    try:  # opt-in NVSwitch reduction, measured for comparison only (not bit-exact)
        if not with_nvls:
            raise RuntimeError("not requested (--nvls)")
        from paper_1811_11141_b200.allreduce_net import enable_nvls

        if not getattr(session, "nvls_bytes", 0):
            enable_nvls(session, max(sizes))
        nvls = _exchange_times(comm, world, device, sizes, kind=4, algo=_native.ALGO_NVLS)
    except Exception as exc:  # unsupported fabric: leave the column out
        print(f"NVLS unavailable: {exc}", file=sys.stderr)
    fused = _exchange_times(comm, world, device, sizes, kind=4)
    # bf16 gradients (fp32 accumulation) at the same payload bytes, vs NCCL bf16
    fused_bf16 = _exchange_times(comm, world, device, sizes, kind=5)
    nccl_bf16 = _nccl_times(world, device, sizes, bf16=True)
    session.raise_if_failed()
    rows = []
    for i, (nbytes, t1, t2, tn) in enumerate(zip(sizes, one, two, nccl)):
        bus = 2 * (world - 1) / world * nbytes
        rows.append({"bytes": nbytes,
                     "oneshot_us": round(t1 * 1e6, 2), "oneshot_busbw_gbs": round(bus / t1 / 1e9, 1),
                     "twoshot_us": round(t2 * 1e6, 2), "twoshot_busbw_gbs": round(bus / t2 / 1e9, 1),
                     "nccl_us": round(tn * 1e6, 2), "nccl_busbw_gbs": round(bus / tn / 1e9, 1),
                     "fused_exchange_us": round(fused[i] * 1e6, 2),
                     "fused_exchange_busbw_gbs": round(bus / fused[i] / 1e9, 1),
                     "fused_bf16_us": round(fused_bf16[i] * 1e6, 2),
                     "fused_bf16_busbw_gbs": round(bus / fused_bf16[i] / 1e9, 1),
                     "nccl_bf16_us": round(nccl_bf16[i] * 1e6, 2),
                     "nccl_bf16_busbw_gbs": round(bus / nccl_bf16[i] / 1e9, 1)})
        if nvls is not None:
            rows[-1]["nvls_fused_us"] = round(nvls[i] * 1e6, 2)
            rows[-1]["nvls_fused_busbw_gbs"] = round(bus / nvls[i] / 1e9, 1)
    return rows


def _fit(sizes, times, world):
    from paper_1811_11141_b200 import CommModel, Measurement, fit_ab

    pts = [(s, t) for s, t in zip(sizes, times) if s <= 32 << 20]
    try:
        return fit_ab([Measurement(s, t, max(world, 2)) for s, t in pts]), True
    except ValueError:  # e.g. under a profiler that serialises launches
        return CommModel(a=min(times), b=0.0), False


def _algo_mix(session, group_bytes):
    """How many groups each AUTO algorithm serves (mirrors the native choice)."""
    import collections

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import _algo_for

    names = {_native.ALGO_LL: "ll", _native.ALGO_ONESHOT: "oneshot", _native.ALGO_TWOSHOT: "twoshot",
             _native.ALGO_PUSH: "push_twoshot", _native.ALGO_PUSH_ONESHOT: "push_oneshot",
             _native.ALGO_PUSH_PIPE: "push_pipe", _native.ALGO_NVLS: "nvls", _native.ALGO_LL128: "ll128_twoshot",
             _native.ALGO_LL128_ONESHOT: "ll128_oneshot"}
    mix = collections.Counter(names.get(_algo_for(session, b // 4, fused=True), "other") for b in group_bytes if b)
    return dict(sorted(mix.items()))


class RankContext:
    """This rank's view of the run: ids, device, communicator and the L2-flush buffer."""

    def __init__(self, rank, world, local, device, comm, session, flush):
        self.rank, self.world, self.local, self.device = rank, world, local, device
        self.comm, self.session, self.flush = comm, session, flush


def run_strategy(ctx, profile, plan, predicted, steps, warmup, *, graph=True, fused=True, keep=False, pdl=True):
    """Warm up, then time `steps` Algorithm-2 iterations of `plan` (max over ranks per
    iteration); every iteration is preceded by an L2 flush outside its events and the
    reduced gradients are verified before and after the timed region."""
    import torch

    from paper_1811_11141_b200.overlap import OverlappedIteration

    world, device = ctx.world, ctx.device
    it = OverlappedIteration(profile, plan, comm=ctx.comm, rank=ctx.rank, world=world, device=device,
                             fill=True, graph=graph, fused=fused, pdl=pdl)
    try:
        for _ in range(warmup):
            with torch.cuda.stream(it.compute_stream):
                l2_flush(ctx.flush)
            it.run()
        if not it.verify():
            raise RuntimeError(f"{profile.name}: reduced gradients differ from the expected sums")
        _barrier(world)
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        t_iter, compute, exposed, kern = [], [], [], []
        for _ in range(steps):
            with torch.cuda.stream(it.compute_stream):
                l2_flush(ctx.flush)  # L2 flush between iterations, outside the iteration's events
            times = it.run()
            t_iter.append(times.t_iter)
            compute.append(times.compute_time)
            exposed.append(times.t_c_no)
            kern.append(it.kernel_times())
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        _barrier(world)
        if ctx.session is not None:
            ctx.session.raise_if_failed()
        ok = it.verify()
        t_iter_max = _max_over_ranks(t_iter, world, device)
        compute_max = _max_over_ranks(compute, world, device)
        exposed_max = _max_over_ranks(exposed, world, device)
        res = {
            "t_iter_ms": round(statistics.fmean(t_iter_max) * 1e3, 4),
            "t_iter_ms_median": round(statistics.median(t_iter_max) * 1e3, 4),
            "t_iter_ms_min": round(min(t_iter_max) * 1e3, 4),
            "compute_ms": round(statistics.fmean(compute_max) * 1e3, 4),
            "t_c_no_us": round(statistics.fmean(exposed_max) * 1e6, 2),
            "t_c_no_us_median": round(statistics.median(exposed_max) * 1e6, 2),
            "scaling_eff": round(statistics.fmean(compute_max) / statistics.fmean(t_iter_max), 5),
            "predicted_t_iter_ms": round(predicted.t_iter * 1e3, 4),
            "predicted_t_c_no_us": round(predicted.t_c_no * 1e6, 2),
            "groups": len(plan.groups()),
            "verified": ok,
            "wall_s": round(wall, 4),
        }
    except BaseException:
        it.close()
        raise
    if not keep:
        it.close()
        it = None
    return res, it, kern, t_iter_max, wall


def pack_unpack_bench(profile, device, flush, hbm_peak, reps=10, warmup=3):
    """Median event-timed K1 pack and K4 unpack of the whole-model bucket (54 rows of one
    contiguous gradient buffer, layer `high` first), each after an L2 flush; algorithmic
    bytes 2 x bucket (read + write).  The kernels AUTO picks here: the TMA bulk path."""
    import ctypes

    import torch

    from paper_1811_11141_b200 import _native

    counts = list(reversed(profile.param_counts()))
    total = sum(counts)
    flat = torch.ones(total, device=device)
    bucket = torch.empty(total, device=device)
    rows, off = [], 0
    for c in counts:
        rows.append((flat[off:off + c].data_ptr(), c, off))
        off += c
    table = _native.DeviceTable(rows)
    stream = torch.cuda.current_stream(device)
    out = {"bytes": 4 * total, "rows": len(rows), "kernel": "bulk_rows_kernel (TMA cp.async.bulk, 4-stage smem ring)",
           "algorithmic_bytes": "2 x bucket bytes per launch", "timing": "one CUDA event pair per launch, "
           "L2 written and read back before each"}
    try:
        for op in ("pack", "unpack"):
            times = []
            for i in range(warmup + reps):
                l2_flush(flush)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if op == "pack":
                    _native.call("mgw_pack", table.ptr, table.n, bucket.data_ptr(), total, ctypes.c_float(1.0),
                                 stream.cuda_stream)
                else:
                    _native.call("mgw_unpack", table.ptr, table.n, bucket.data_ptr(), total, stream.cuda_stream)
                b.record(stream)
                b.synchronize()
                if i >= warmup:
                    times.append(a.elapsed_time(b) * 1e-3)
            t = statistics.median(times)
            gbs = 2 * 4 * total / t / 1e9
            out[op] = {"us": round(t * 1e6, 2), "achieved": round(gbs, 1), "frac": round(gbs / hbm_peak, 4)}
        out["round_trip_exact"] = bool(torch.equal(flat, torch.ones_like(flat)))
    finally:
        table.close()
    traffic_file = ROOT / "profiles" / "roofline_traffic.json"
    if traffic_file.exists():
        doc = json.loads(traffic_file.read_text())
        out["traffic"] = {op: doc.get(f"K1 pack@102MB" if op == "pack" else "K4 unpack@102MB") for op in ("pack", "unpack")}
    return out


def run_ours(args) -> dict | None:
    import torch

    from paper_1811_11141_b200 import (
        CommModel,
        Measurement,
        MergePlan,
        find_merge_plan,
        fit_ab,
        simulate_mgwfbp,
        simulate_sync_easgd,
        simulate_wfbp,
    )
    from paper_1811_11141_b200.allreduce_net import open_session_dist
    from paper_1811_11141_b200.overlap import OverlappedIteration

    rank, world, local = _dist_setup(args)
    device = torch.device("cuda", local)
    profile, bwd, fwd = b200_profile()
    n = profile.num_layers
    session = comm = None
    if world > 1:
        _, session = open_session_dist(capacity_bytes=4 * profile.total_params)
        comm = session.comm

    # 1. fit the startup/bandwidth model of one group exchange on this box
    exch = _exchange_times(comm, world, device, FIT_SIZES, kind=0 if args.unfused else 4,
                           repeats=3 if args.quick else 20, warmups=1 if args.quick else 3)
    # the same exchange steps replayed as one CUDA graph: the per-launch cost inside the
    # engine's graph (reported next to the stream-timed fit the planner uses)
    exch_graph = _exchange_times(comm, world, device, FIT_SIZES,
                                 kind=(0 if args.unfused else 4) | 256, repeats=3 if args.quick else 20,
                                 warmups=1 if args.quick else 3)
    if session is not None:
        session.raise_if_failed()
    model, fit_ok = _fit(FIT_SIZES, exch, world)
    model_graph, _ = _fit(FIT_SIZES, exch_graph, world)
    plans = {
        "wfbp": MergePlan(frozenset(), n),
        "synceasgd": MergePlan(frozenset(range(2, n + 1)), n),
        "mgwfbp": find_merge_plan(profile, model),
    }
    predicted = {
        "wfbp": simulate_wfbp(profile, model),
        "synceasgd": simulate_sync_easgd(profile, model),
        "mgwfbp": simulate_mgwfbp(profile, model, plans["mgwfbp"]),
    }

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=device)
    ctx = RankContext(rank, world, local, device, comm, session, flush)
    results = {}
    headline = None
    for name in ("wfbp", "synceasgd", "mgwfbp"):
        sampler = ClockSampler(local) if (rank == 0 and name == "mgwfbp") else None
        if sampler:
            sampler.__enter__()
        res, it, kern, t_iter_max, wall = run_strategy(ctx, profile, plans[name], predicted[name], args.steps,
                                                        args.warmup, graph=not args.no_graph,
                                                        fused=not args.unfused, keep=name == "mgwfbp",
                                                        pdl=not args.no_pdl)
        results[name] = res
        if name == "mgwfbp":
            headline = (it, kern, it.group_bytes(), sampler, t_iter_max, wall)
            launches = it.launches_per_iteration

    it, kern, gbytes, sampler, t_iter_max, wall = headline
    # roofline of the dominant kernel inside the MG-WFBP timed region; kernel spans are
    # %globaltimer stamps written by the kernels (first CTA entry .. last CTA exit)
    steps = len(kern)
    fused = not args.unfused
    if fused:  # one kernel per group (N = 1: pack -> one-input fold -> write-back)
        spans = {"fused": sum(sum(k[1]) for k in kern)}
    else:
        spans = {"pack": sum(sum(k[0]) for k in kern), "unpack": sum(sum(k[2]) for k in kern)}
        if world > 1:
            spans["allreduce"] = sum(sum(k[1]) for k in kern)
    dominant = max(spans, key=spans.get)
    total_bytes = sum(gbytes)
    sending = sum(1 for b in gbytes if b)
    hbm_peak, hbm_src = peaks()
    names = {"pack": "K1 pack", "unpack": "K4 unpack", "allreduce": "K2/K3 all-reduce",
             "fused": "fused K1+K4 (N=1)" if world == 1 else "fused K1+K2/K3+K4"}
    n1_note = ("N=1 has nothing to exchange: the group kernel runs as the stand-in of the N>1 exchange "
               "(pack -> one-input fold -> write-back per group, the exchange's local HBM legs) so every N "
               "runs the same per-group launch schedule; its small groups are launch/latency-bound")
    if world == 1 or dominant in ("pack", "unpack"):
        # HBM: pack / unpack read + write every bucket byte once; the N=1 fused kernel does both
        per_unit = 4 if dominant == "fused" else 2
        per_step = per_unit * total_bytes
        achieved = per_step * steps / spans[dominant] / 1e9
        roofline = {"bound": "hbm", "kernel": names[dominant],
                    "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(achieved / hbm_peak, 4), "peak_source": hbm_src,
                    "algorithmic_bytes": f"{per_unit} x group bucket bytes per launch"}
        if world == 1 and dominant == "fused":
            roofline["note"] = n1_note
    else:
        per_unit = 2 * (world - 1) / world
        per_step = int(per_unit * total_bytes)  # nccl-tests bus bytes
        achieved = per_step * steps / spans[dominant] / 1e9
        roofline = {"bound": "nvlink", "kernel": names[dominant],
                    "achieved": round(achieved, 1),
                    "peak": NVLINK_PEAK_GBS, "unit": "GB/s", "frac": round(achieved / NVLINK_PEAK_GBS, 4),
                    "peak_source": "measured peer copy per direction, B200_PROFILING.md (900 nominal)",
                    "algorithmic_bytes": "2(N-1)/N x group bucket bytes per launch (bus bytes)",
                    "bound_note": "a collective is bound by the NVLink fabric, neither HBM nor tensor cores; "
                                  "peak = the per-GPU peer-copy bandwidth of B200_PROFILING.md"}
    roofline.update({
        "bytes_per_step": per_step,
        "launches_per_step": sending,
        "avg_launch_us": round(spans[dominant] / (steps * max(1, sending)) * 1e6, 3),
        "timing": "kernel-written %globaltimer spans over the timed region (CUDA event records cost ~6.5 us "
                  "per pair inside a graph on this B200, see profiles/microbench_r01.json)",
        "kernel_ms_per_step": {k: round(v / steps * 1e3, 4) for k, v in spans.items()},
    })
    traffic_file = ROOT / "profiles" / "roofline_traffic.json"
    roofline["traffic"] = None
    if traffic_file.exists():
        roofline["traffic"] = json.loads(traffic_file.read_text()).get(f"{roofline['kernel']}@N{world}")
    # the same kernel on the whole-model bucket, back to back under one event pair
    big_kind = {"pack": 2, "allreduce": 1, "unpack": 3, "fused": 4}[dominant]
    big = _exchange_times(comm, world, device, [4 * profile.total_params], kind=big_kind)[0]
    big_bw = per_unit * 4 * profile.total_params / big / 1e9
    roofline["whole_model_bucket"] = {"bytes": 4 * profile.total_params, "us": round(big * 1e6, 2),
                                      "achieved": round(big_bw, 1),
                                      "frac": round(big_bw / (hbm_peak if roofline["bound"] == "hbm" else NVLINK_PEAK_GBS), 4),
                                      "timing": "one CUDA event pair around 20 back-to-back launches"}
    # K1 pack / K4 unpack alone on the whole-model bucket (the SyncEASGD group), each launch
    # timed by its own event pair after an L2 flush: the HBM-bound kernels at full size
    if world == 1:
        roofline["pack_unpack_whole_model"] = pack_unpack_bench(profile, device, flush, hbm_peak)

    # e2e: the same MG-WFBP iteration with host buffers (H2D of every layer's gradient,
    # D2H of every reduced gradient) inside the timed region
    if args.quick:
        args.no_sweep = args.no_cpu_baseline = True
    e2e_it = OverlappedIteration(profile, plans["mgwfbp"], comm=comm, rank=rank, world=world, device=device,
                                 host_io=True, graph=not args.no_graph, fused=not args.unfused)
    try:
        for _ in range(args.warmup):
            e2e_it.run()
        _barrier(world)
        e2e_times = []
        for _ in range(args.steps):
            with torch.cuda.stream(e2e_it.compute_stream):
                l2_flush(flush)
            e2e_times.append(e2e_it.run().t_iter)
        e2e_ok = e2e_it.verify()
        h2d, d2h = e2e_it.io_bytes()
    finally:
        e2e_it.close()
    e2e_max = _max_over_ranks(e2e_times, world, device)
    if sampler is not None:
        sampler.__exit__(None, None, None)

    sweep = None
    if world > 1 and not args.no_sweep:
        sweep = _allreduce_sweep(session, comm, world, device, FIT_SIZES, with_nvls=args.nvls)
    it.close()
    if session is not None:
        session.close()
    if rank != 0:
        return None

    mg = results["mgwfbp"]
    same_as_wfbp = plans["mgwfbp"].merged_layers == plans["wfbp"].merged_layers
    line = {
        "metric": METRIC,
        "value": mg["t_iter_ms"],
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": mg["t_iter_ms"],
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": "synthetic (reference gradient pattern rank+1+layer%5, rewritten every iteration)",
        "config": workload_config(bwd, fwd, world),
        "run": {
            "plan_groups": len(plans["mgwfbp"].groups()),
            "merged_layers": sorted(plans["mgwfbp"].merged_layers),
            "fitted_a_us": round(model.a * 1e6, 3),
            "fitted_b_ns_per_byte": model.b * 1e9,
            "fit_ok": fit_ok,
            "fitted_a_graph_us": round(model_graph.a * 1e6, 3),
            "fitted_b_graph_ns_per_byte": model_graph.b * 1e9,
            "cuda_graph": not args.no_graph,
            "fused_group_kernel": not args.unfused,
            "programmatic_launch": not args.no_pdl,
            "group_algorithms": _algo_mix(session, gbytes) if (session is not None and not args.unfused) else None,
        },
        "strategies": results,
        "mgwfbp_plan_equals_wfbp": same_as_wfbp,
        "roofline": roofline,
        "e2e": {"value": round(statistics.fmean(e2e_max) * 1e3, 4), "unit": "ms",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "verified": e2e_ok},
        "gpu_launches": launches * args.steps,
        "group_exchange_us": {str(s): round(t * 1e6, 2) for s, t in zip(FIT_SIZES, exch)},
        "group_exchange_graph_us": {str(s): round(t * 1e6, 2) for s, t in zip(FIT_SIZES, exch_graph)},
        "timed_wall_s": round(wall, 4),
    }
    if sweep is not None:
        line["allreduce_sweep"] = sweep
    if sampler is not None:
        line["clocks"] = sampler.summary()
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(profile, plans["mgwfbp"], world, args.cpu_seconds)
    return line


# --------------------------------------------------------- reference arm (CPU)


def _cpu_plan(profile, n_ranks):
    """The reference workflow on its own transport: fit (a, b) on the CPU ring, plan."""
    from oracle import emulation
    from paper_1811_11141_b200 import Measurement, MergePlan, find_merge_plan, fit_ab

    if n_ranks < 2:
        return MergePlan(frozenset(), profile.num_layers), None
    sizes = [1 << k for k in range(14, 25, 2)]
    ms = [Measurement(s, emulation.ring_seconds(n_ranks, s, repeats=3), n_ranks) for s in sizes]
    model = fit_ab(ms)
    return find_merge_plan(profile, model), model


def cpu_baseline(profile, plan, n_ranks, seconds):
    from oracle import emulation

    walls, ok = emulation.emulate(profile, plan, n_ranks, 10_000, warmup=1, time_budget_s=seconds)
    host_cores, cpu_model = host_cpu()
    return {
        "value": round(statistics.fmean(walls) * 1e3, 3),
        "unit": "ms",
        "cores": max(1, n_ranks),
        "host_cores": host_cores,
        "cpu_model": cpu_model,
        "kind": "port",
        "sample": f"{len(walls)} Algorithm-2 iterations of the same resnet50_like profile/plan with {n_ranks} "
                  f"simulated rank(s) (oracle/emulation.py: reference _delay + C ring, one thread per rank), "
                  f"~{seconds:.0f} s budget, verified={ok}",
    }


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    profile, bwd, fwd = b200_profile()
    n_ranks = args.gpus
    plan, model = _cpu_plan(profile, n_ranks)
    from oracle import emulation

    _, _ = emulation.emulate(profile, plan, n_ranks, args.warmup, warmup=0)
    t0 = time.perf_counter()
    walls, ok = emulation.emulate(profile, plan, n_ranks, args.steps, warmup=0,
                                  time_budget_s=max(10.0, args.cpu_seconds))
    wall = time.perf_counter() - t0
    value = round(statistics.fmean(walls) * 1e3, 3)
    cores = max(1, n_ranks)
    host_cores, cpu_model = host_cpu()
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "ms",
        "n_gpus": args.gpus,
        "steps": len(walls),
        "warmup": args.warmup,
        "ms_per_step": value,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": "synthetic (reference gradient pattern rank+1+layer%5)",
        "config": workload_config(bwd, fwd, n_ranks),
        "run": {
            "plan_groups": len(plan.groups()),
            "fitted_a_us": None if model is None else round(model.a * 1e6, 3),
            "fitted_b_ns_per_byte": None if model is None else model.b * 1e9,
            "ranks": f"{n_ranks} simulated ranks on host cores (one thread each)",
        },
        "cpu_baseline": {"value": value, "unit": "ms", "cores": cores, "host_cores": host_cores,
                         "cpu_model": cpu_model, "kind": "port",
                         "sample": f"{len(walls)} iterations, {n_ranks} simulated rank(s), oracle/emulation.py "
                                   f"(reference Algorithm 2: _delay agent thread + C ring one thread per rank), "
                                   f"verified={ok}, wall {wall:.1f} s"},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-graph", action="store_true", help="eager stream schedule instead of CUDA-graph replay")
    ap.add_argument("--unfused", action="store_true", help="separate pack / all-reduce / unpack kernels per group")
    ap.add_argument("--no-pdl", action="store_true",
                    help="launch each group's exchange after its gradient fill completes (no programmatic launch)")
    ap.add_argument("--nvls", action="store_true", help="also time the opt-in NVLS exchange in the sweep (N > 1)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the all-reduce bus-bandwidth sweep (N > 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--quick", action="store_true",
                    help="profiling aid: 3 fit repetitions, no e2e / sweep / CPU baseline")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    # keep stdout for the one JSON line: library chatter (e.g. "NCCL version") goes to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    try:
        line = run_reference(args) if args.impl == "reference" else run_ours(args)
    finally:
        sys.stdout.flush()
        os.dup2(json_fd, 1)
        os.close(json_fd)
    if line is not None:
        print(json.dumps(line), flush=True)
    if args.impl == "ours" and args.gpus > 1:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
