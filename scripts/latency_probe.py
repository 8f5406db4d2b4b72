"""Small-message latency breakdown over the real IPC path (torchrun, one rank per GPU).

    torchrun --nproc-per-node N scripts/latency_probe.py

Loop-timed (mgw_time_exchange: 50 back-to-back steps under one CUDA event pair, max over
ranks) for 4 KiB .. 1 MiB: the gate rendezvous alone (kind 6: one-warp fabric round trip
+ a counter kernel), the fused exchange per algorithm (LL / one-shot / two-shot), the
bare all-reduce kernels, the bf16 exchange, and a local pack (launch floor).
"""

from __future__ import annotations

import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    import torch

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    class A:
        gpus = int(os.environ.get("WORLD_SIZE", "1"))

    rank, world, local = bench._dist_setup(A())
    device = torch.device("cuda", local)
    _, session = open_session_dist(capacity_bytes=64 << 20)
    comm = session.comm
    sizes = [4096, 16384, 65536, 262144, 1 << 20]
    def T(limit=None, **kw):
        ok = [m for m in sizes if limit is None or m <= limit]
        got = [round(t * 1e6, 2) for t in bench._exchange_times(comm, world, device, ok, repeats=50, **kw)]
        return got + [None] * (len(sizes) - len(ok))

    out = {"world": world, "sizes": sizes, "us": {
        "gate_plus_counter": T(kind=6),
        "fused_ll": T(kind=4, algo=_native.ALGO_LL, limit=262144),
        "fused_oneshot": T(kind=4, algo=_native.ALGO_ONESHOT),
        "fused_twoshot": T(kind=4, algo=_native.ALGO_TWOSHOT),
        "allreduce_oneshot": T(kind=1, algo=_native.ALGO_ONESHOT),
        "allreduce_twoshot": T(kind=1, algo=_native.ALGO_TWOSHOT),
        "fused_bf16_auto": T(kind=5),
        "local_pack": [round(t * 1e6, 2) for t in bench._exchange_times(None, 1, device, sizes, kind=2, repeats=50)],
        # the same steps replayed as one CUDA graph (kind | MGW_TIME_GRAPH): engine-like launch cost
        "graph_fused_ll": T(kind=4 | 256, algo=_native.ALGO_LL, limit=262144),
        "graph_fused_auto": T(kind=4 | 256),
        "graph_gate_plus_counter": T(kind=6 | 256),
        "graph_local_pack": [round(t * 1e6, 2) for t in
                             bench._exchange_times(None, 1, device, sizes, kind=2 | 256, repeats=50)],
    }}
    # CTA-count sensitivity of the fused one-shot (16-B slots per CTA; default 512 x Unroll)
    for per in (128, 256, 512):
        _native.call("mgw_comm_set_tuning", comm, 0, per)
        out["us"][f"fused_oneshot_per{per}"] = T(kind=4, algo=_native.ALGO_ONESHOT)
    _native.call("mgw_comm_set_tuning", comm, 0, 0)
    for per in (256, 512):
        _native.call("mgw_comm_set_tuning", comm, 1, per)
        out["us"][f"fused_twoshot_per{per}"] = T(kind=4, algo=_native.ALGO_TWOSHOT)
    _native.call("mgw_comm_set_tuning", comm, 1, 0)
    session.raise_if_failed()
    session.close()
    if rank == 0:
        print(json.dumps(out))
    import torch.distributed as dist

    dist.destroy_process_group()


if __name__ == "__main__":
    main()
