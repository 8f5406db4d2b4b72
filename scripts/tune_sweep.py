"""Tuning sweep (torchrun): CTA work size and CTA cap for the one-shot / two-shot /
fused kernels over a size range; prints one JSON document on rank 0."""

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
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    device = torch.device("cuda", local)
    sizes = [1 << k for k in range(18, 28)]
    _, session = open_session_dist(capacity_bytes=max(sizes))
    comm = session.comm
    res = {}
    for ctas in (148, 296):
        _native.call("mgw_comm_set_max_ctas", comm, ctas)
        for per in (0, 256, 512, 2048):
            _native.call("mgw_comm_set_tuning", comm, 0, per)
            _native.call("mgw_comm_set_tuning", comm, 1, per)
            res[f"one_c{ctas}_p{per}"] = bench._exchange_times(comm, world, device, sizes, kind=1, algo=_native.ALGO_ONESHOT)
            res[f"two_c{ctas}_p{per}"] = bench._exchange_times(comm, world, device, sizes, kind=1, algo=_native.ALGO_TWOSHOT)
            res[f"fusedtwo_c{ctas}_p{per}"] = bench._exchange_times(comm, world, device, sizes, kind=4, algo=_native.ALGO_TWOSHOT)
            res[f"fusedone_c{ctas}_p{per}"] = bench._exchange_times(comm, world, device, sizes, kind=4, algo=_native.ALGO_ONESHOT)
    res["nccl"] = bench._nccl_times(world, device, sizes)
    session.raise_if_failed()
    session.close()
    if rank == 0:
        out = {"world": world, "sizes": sizes, "us": {k: [round(x * 1e6, 2) for x in v] for k, v in res.items()}}
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
