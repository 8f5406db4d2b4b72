"""Bus GB/s of each fused group exchange algorithm vs size, next to ncclAllReduce (torchrun,
one rank per GPU): device time per exchange from mgw_time_exchange (kind 4, `reps` back to
back under one event pair; graph mode = the reps replayed as one CUDA graph, the engine's
way), max over ranks.  Bus bytes = 2 (N-1)/N x M (nccl-tests convention).

    torchrun --nproc-per-node N scripts/algo_sweep.py [--mib 4,8,16,32,64,128]
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", default="1,4,8,16,32,64,128")
    ap.add_argument("--algos", default="twoshot,push,push_pipe,auto")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--pipe-subs", default="", help="comma list of pipelined sub-chunk slots to sweep")
    ap.add_argument("--bf16", action="store_true", help="bf16 gradients (fp32 accumulation) vs NCCL bf16")
    ap.add_argument("--max-ctas", default="", help="comma list of CTA caps to sweep for the listed algorithms")
    ap.add_argument("--per-cta", default="", help="comma list of two-shot / push slots per CTA to sweep")
    ap.add_argument("--per-cta-algos", default="", help="algorithms of the --per-cta sweep (default: --algos)")
    args = ap.parse_args()
    import torch

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    class A:
        gpus = int(os.environ.get("WORLD_SIZE", "1"))

    rank, world, local = bench._dist_setup(A())
    device = torch.device("cuda", local)
    sizes = [int(float(m) * (1 << 20)) for m in args.mib.split(",")]
    # the one-shot kinds hold N incoming rows of the whole bucket (LL128: in 128-B lines of 112 B)
    _, session = open_session_dist(capacity_bytes=max(sizes) * world * 8 // 7 + (1 << 20))
    comm = session.comm
    ids = {"oneshot": _native.ALGO_ONESHOT, "twoshot": _native.ALGO_TWOSHOT, "push": _native.ALGO_PUSH,
           "push_pipe": _native.ALGO_PUSH_PIPE, "push_oneshot": _native.ALGO_PUSH_ONESHOT, "auto": _native.ALGO_AUTO,
           "ll128": _native.ALGO_LL128, "ll128_one": _native.ALGO_LL128_ONESHOT, "ll": _native.ALGO_LL}
    out = {"world": world, "sizes": sizes, "bus_gbs": {}, "us": {}}
    for name in args.algos.split(","):
        for graph in (False, True):
            kind = (5 if args.bf16 else 4) | (256 if graph else 0)
            t = bench._exchange_times(comm, world, device, sizes, kind=kind, algo=ids[name], repeats=args.reps)
            key = name + ("@graph" if graph else "@stream")
            out["us"][key] = [round(x * 1e6, 2) for x in t]
            out["bus_gbs"][key] = [round(2 * (world - 1) / world * s / x / 1e9, 1) for s, x in zip(sizes, t)]
    if args.max_ctas:
        _native.call("mgw_set_option", _native.OPT_WIDE_MIN_BYTES, 0)  # the cap as given
    for cap in [int(v) for v in args.max_ctas.split(",") if v]:
        _native.call("mgw_comm_set_max_ctas", comm, cap)
        for name in args.algos.split(","):
            t = bench._exchange_times(comm, world, device, sizes, kind=(5 if args.bf16 else 4) | 256, algo=ids[name],
                                      repeats=args.reps)
            key = f"{name}_cap{cap}@graph"
            out["us"][key] = [round(x * 1e6, 2) for x in t]
            out["bus_gbs"][key] = [round(2 * (world - 1) / world * s / x / 1e9, 1) for s, x in zip(sizes, t)]
    _native.call("mgw_comm_set_max_ctas", comm, 296)
    _native.call("mgw_set_option", _native.OPT_WIDE_MIN_BYTES, 112 << 20)
    for per in [int(v) for v in args.per_cta.split(",") if v]:
        _native.call("mgw_comm_set_tuning", comm, 1, per)
        for name in (args.per_cta_algos or args.algos).split(","):
            t = bench._exchange_times(comm, world, device, sizes, kind=(5 if args.bf16 else 4) | 256, algo=ids[name],
                                      repeats=args.reps)
            key = f"{name}_per{per}@graph"
            out["us"][key] = [round(x * 1e6, 2) for x in t]
            out["bus_gbs"][key] = [round(2 * (world - 1) / world * s / x / 1e9, 1) for s, x in zip(sizes, t)]
    _native.call("mgw_comm_set_tuning", comm, 1, 0)
    for slots in [int(v) for v in args.pipe_subs.split(",") if v]:
        _native.call("mgw_set_option", _native.OPT_PIPE_SUB_SLOTS, slots)
        t = bench._exchange_times(comm, world, device, sizes, kind=4 | 256, algo=_native.ALGO_PUSH_PIPE,
                                  repeats=args.reps)
        key = f"push_pipe_sub{slots}@graph"
        out["us"][key] = [round(x * 1e6, 2) for x in t]
        out["bus_gbs"][key] = [round(2 * (world - 1) / world * s / x / 1e9, 1) for s, x in zip(sizes, t)]
    _native.call("mgw_set_option", _native.OPT_PIPE_SUB_SLOTS, 512)
    nccl = bench._nccl_times(world, device, sizes, repeats=args.reps, bf16=args.bf16)
    out["us"]["nccl@stream"] = [round(x * 1e6, 2) for x in nccl]
    out["bus_gbs"]["nccl@stream"] = [round(2 * (world - 1) / world * s / x / 1e9, 1) for s, x in zip(sizes, nccl)]
    session.raise_if_failed()
    session.close()
    if rank == 0:
        print(json.dumps(out))
    import torch.distributed as dist

    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
