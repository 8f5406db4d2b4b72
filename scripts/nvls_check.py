"""NVLS (opt-in) check and timing under torchrun: fused NVLS exchange vs the exact sum
(tolerance) and vs the bit-exact two-shot; prints one JSON document on rank 0, exits 1
on a tolerance failure.

    torchrun --nproc-per-node N scripts/nvls_check.py
"""

from __future__ import annotations

import ctypes
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import enable_nvls, open_session_dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    cap = 256 << 20
    _, session = open_session_dist(capacity_bytes=cap)
    enable_nvls(session, cap)
    comm = session.comm
    s = torch.cuda.current_stream()
    worst = 0.0
    identical = True
    for n in (1, 17, 4099, 65537, 1 << 20, (1 << 24) + 3):
        g = torch.Generator(device=dev).manual_seed(n * 31 + rank)
        x = torch.randn(n, device=dev, generator=g)
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x)
        exact = torch.stack([p.double() for p in parts]).sum(0)
        bound = torch.stack([p.double().abs() for p in parts]).sum(0) * world * 2.0 ** -24
        table = _native.DeviceTable([(x.data_ptr(), n, 0)])
        _native.call("mgw_allreduce_fused", comm, table.ptr, 1, n, ctypes.c_float(1.0), _native.ALGO_NVLS, s.cuda_stream)
        torch.cuda.synchronize()
        session.raise_if_failed()
        table.close()
        err = (x.double() - exact).abs()
        worst = max(worst, float((err / bound.clamp_min(1e-300)).max()))
        lo, hi = x.clone(), x.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        identical = identical and bool(torch.equal(lo, hi))
    sizes = [1 << k for k in range(20, 28)]
    nvls = bench._exchange_times(comm, world, dev, sizes, kind=4, algo=_native.ALGO_NVLS)
    two = bench._exchange_times(comm, world, dev, sizes, kind=4, algo=_native.ALGO_TWOSHOT)
    nccl = bench._nccl_times(world, dev, sizes)
    rows = []
    for b, t1, t2, t3 in zip(sizes, nvls, two, nccl):
        bus = 2 * (world - 1) / world * b
        rows.append({"bytes": b, "nvls_fused_us": round(t1 * 1e6, 2), "nvls_fused_busbw": round(bus / t1 / 1e9, 1),
                     "twoshot_fused_us": round(t2 * 1e6, 2), "twoshot_fused_busbw": round(bus / t2 / 1e9, 1),
                     "nccl_us": round(t3 * 1e6, 2), "nccl_busbw": round(bus / t3 / 1e9, 1)})
    session.close()
    ok = worst <= 1.0 and identical
    if rank == 0:
        print(json.dumps({"world": world, "worst_error_over_bound": worst, "ranks_identical": identical, "ok": ok,
                          "rows": rows}))
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
