"""NVLS (opt-in) grid sensitivity vs the push two-shot, engine mode (graph replay),
large buckets.  torchrun --nproc-per-node N scripts/nvls_tune.py"""

from __future__ import annotations

import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    import torch
    import torch.distributed as dist

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import enable_nvls, open_session_dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    cap = (128 << 20) + (1 << 20)
    _, session = open_session_dist(capacity_bytes=cap)
    enable_nvls(session, 128 << 20)
    comm = session.comm
    sizes = [16 << 20, 32 << 20, 64 << 20, 128 << 20]
    out = {"world": world, "sizes": sizes, "us": {}}
    out["us"]["push_default"] = [round(x * 1e6, 2) for x in bench._exchange_times(
        comm, world, dev, sizes, kind=4 | 256, algo=_native.ALGO_PUSH)]
    for cap_ctas in (148, 296, 512):
        _native.call("mgw_comm_set_max_ctas", comm, cap_ctas)
        for per in (0, 4096, 8192):
            _native.call("mgw_comm_set_tuning", comm, 1, per)
            t = bench._exchange_times(comm, world, dev, sizes, kind=4 | 256, algo=_native.ALGO_NVLS)
            out["us"][f"nvls_cap{cap_ctas}_per{per or 'dflt'}"] = [round(x * 1e6, 2) for x in t]
    _native.call("mgw_comm_set_tuning", comm, 1, 0)
    _native.call("mgw_comm_set_max_ctas", comm, 296)
    session.raise_if_failed()
    for k, v in list(out["us"].items()):
        out["us"][k + "_busbw"] = [round(2 * (world - 1) / world * s / (t * 1e-6) / 1e9, 1) for s, t in zip(sizes, v)]
    session.close()
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
