"""All-reduce bus-bandwidth sweep (torchrun, one rank per GPU): our one-shot and
two-shot kernels at several CTA caps, the full group exchange, and ncclAllReduce.

    torchrun --nproc-per-node N scripts/ar_sweep.py [--ctas 148,296] [--sizes ...]
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", default="296")
    ap.add_argument("--sizes", default=",".join(str(1 << k) for k in range(12, 28)))
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    device = torch.device("cuda", local)
    sizes = [int(x) for x in args.sizes.split(",")]
    _, session = open_session_dist(capacity_bytes=max(sizes))
    comm = session.comm
    out = {"world": world, "rows": []}
    res = {}
    for ctas in [int(c) for c in args.ctas.split(",")]:
        _native.call("mgw_comm_set_max_ctas", comm, ctas)
        for algo, name in ((_native.ALGO_ONESHOT, "oneshot"), (_native.ALGO_TWOSHOT, "twoshot")):
            res[f"{name}_{ctas}"] = bench._exchange_times(comm, world, device, sizes, kind=1, algo=algo, repeats=args.reps)
        res[f"exchange_{ctas}"] = bench._exchange_times(comm, world, device, sizes, kind=0, repeats=args.reps)
        res[f"fused_{ctas}"] = bench._exchange_times(comm, world, device, sizes, kind=4, repeats=args.reps)
        _native.call("mgw_comm_set_ll_max", comm, 0)
        res[f"fused_noll_{ctas}"] = bench._exchange_times(comm, world, device, sizes, kind=4, repeats=args.reps)
        _native.call("mgw_comm_set_ll_max", comm, 256 << 10)
        res[f"fused_ll256k_{ctas}"] = bench._exchange_times(comm, world, device, [s for s in sizes], kind=4, repeats=args.reps)
        _native.call("mgw_comm_set_ll_max", comm, 64 << 10)
    res["nccl"] = bench._nccl_times(world, device, sizes, repeats=args.reps)
    session.raise_if_failed()
    for i, nbytes in enumerate(sizes):
        bus = 2 * (world - 1) / world * nbytes
        row = {"bytes": nbytes}
        for k, v in res.items():
            row[k + "_us"] = round(v[i] * 1e6, 2)
            row[k + "_gbs"] = round(bus / v[i] / 1e9, 1)
        out["rows"].append(row)
    session.close()
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
