"""Where the time of one group exchange goes, per algorithm and size (torchrun, one rank
per GPU): the kernels' own %globaltimer marks (mgw_probe_phases) -- ncu cannot replay a
multi-rank kernel.  Median over reps of CTA 0's phase durations, plus the whole-kernel
span (first CTA entry -> last CTA exit), max over ranks.

    torchrun --nproc-per-node N scripts/phase_probe.py
"""

from __future__ import annotations

import ctypes
import json
import os
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402

PHASES = {
    "ll": ["push", "header", "fold"],
    "oneshot": ["pack", "barrier", "remote_fold"],
    "push1": ["push", "barrier", "local_fold"],
    "twoshot": ["pack", "barrier1", "remote_reduce", "barrier2", "remote_gather"],
    "push": ["push_parts", "barrier1", "fold_push", "barrier2", "local_unpack"],
}


def main():
    import torch

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    class A:
        gpus = int(os.environ.get("WORLD_SIZE", "1"))

    rank, world, local = bench._dist_setup(A())
    device = torch.device("cuda", local)
    _, session = open_session_dist(capacity_bytes=(64 << 20) + (1 << 20))
    comm = session.comm
    algos = {"ll": _native.ALGO_LL, "oneshot": _native.ALGO_ONESHOT, "push1": _native.ALGO_PUSH_ONESHOT,
             "twoshot": _native.ALGO_TWOSHOT, "push": _native.ALGO_PUSH}
    sizes = [4096, 65536, 262144, 1 << 20, 4 << 20, 16 << 20]
    reps = 20
    buf = torch.ones((16 << 20) // 4, device=device)
    stream = torch.cuda.Stream(device=device)
    out = {"world": world, "sizes": sizes, "us": {}}
    for name, algo in algos.items():
        for nbytes in sizes:
            if name == "ll" and nbytes > 262144:
                continue
            n = nbytes // 4
            table = _native.DeviceTable([(buf.data_ptr(), n, 0)])
            marks = (ctypes.c_uint64 * (reps * 8))()
            _native.call("mgw_probe_phases", comm, table.ptr, 1, n, algo, reps, marks, stream.cuda_stream)
            table.close()
            rows = [list(marks[r * 8:(r + 1) * 8]) for r in range(2, reps)]  # drop two warm-ups
            k = len(PHASES[name])
            med = lambda xs: statistics.median(xs)  # noqa: E731
            phases = [med([(r[3 + i] - r[2 + i]) * 1e-3 for r in rows]) for i in range(k)]
            span = med([(r[1] - r[0]) * 1e-3 for r in rows])
            vals = bench._max_over_ranks(phases + [span], world, device)
            out["us"][f"{name}@{nbytes}"] = {**{p: round(v, 2) for p, v in zip(PHASES[name], vals[:k])},
                                              "kernel_span": round(vals[k], 2)}
    session.raise_if_failed()
    session.close()
    if rank == 0:
        print(json.dumps(out, indent=1))
    import torch.distributed as dist

    dist.destroy_process_group()


if __name__ == "__main__":
    main()
