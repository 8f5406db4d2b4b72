"""Grid-size sensitivity of the fused group exchange in the engine's mode (graph replay),
mid-size buckets (the ResNet-50 layer range): 16-B slots per CTA x CTA cap, per algorithm.

    torchrun --nproc-per-node N scripts/grid_sweep.py
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
    _, session = open_session_dist(capacity_bytes=(128 << 20) + (1 << 20))
    comm = session.comm
    sizes = [65536, 131072, 262144, 524288, 1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20]
    if os.environ.get("GRID_LARGE"):
        sizes = [8 << 20, 16 << 20, 32 << 20, 64 << 20, 128 << 20]
    out = {"world": world, "sizes": sizes, "us": {}}
    # defaults of every fused algorithm, engine mode (graph replay) and stream mode
    for name, algo in (("ll", _native.ALGO_LL), ("one", _native.ALGO_ONESHOT), ("two", _native.ALGO_TWOSHOT),
                       ("push", _native.ALGO_PUSH), ("push1", _native.ALGO_PUSH_ONESHOT), ("auto", _native.ALGO_AUTO)):
        ok = [m for m in sizes if name != "ll" or m <= (1 << 20)]
        for mode, flag in (("graph", 256), ("stream", 0)):
            t = bench._exchange_times(comm, world, device, ok, kind=4 | flag, algo=algo, repeats=20)
            out["us"][f"{name}_default_{mode}"] = [round(x * 1e6, 2) for x in t] + [None] * (len(sizes) - len(ok))
    if os.environ.get("GRID_DEFAULTS_ONLY"):
        sweep = ()
    elif os.environ.get("GRID_PUSH_ONLY"):
        sweep = ((_native.ALGO_PUSH, 1, "push"),)
    else:
        sweep = ((_native.ALGO_ONESHOT, 0, "one"), (_native.ALGO_TWOSHOT, 1, "two"))
    for algo, key, name in sweep:
        caps = (148, 296, 512)
        pers = (128, 256, 512, 0) if name != "push" else (512, 1024, 2048, 4096, 0)
        for cap in caps:
            _native.call("mgw_comm_set_max_ctas", comm, cap)
            for per in pers:
                _native.call("mgw_comm_set_tuning", comm, key, per)
                t = bench._exchange_times(comm, world, device, sizes, kind=4 | 256, algo=algo, repeats=20)
                out["us"][f"{name}_cap{cap}_per{per or 'dflt'}"] = [round(x * 1e6, 2) for x in t]
            _native.call("mgw_comm_set_tuning", comm, key, 0)
    _native.call("mgw_comm_set_max_ctas", comm, 296)
    session.raise_if_failed()
    session.close()
    if rank == 0:
        print(json.dumps(out))
    import torch.distributed as dist

    dist.destroy_process_group()


if __name__ == "__main__":
    main()
