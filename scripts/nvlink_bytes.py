"""NVLink payload bytes per exchange, measured by the NVLink counters (NVML field values
NVLINK_THROUGHPUT_DATA_TX / _RX, summed over all links, KiB) around `reps` back-to-back
fused group exchanges of M bytes per algorithm -- checked against the byte accounting the
session reports (TransportCounters; the reference pins per-rank payload bytes,
test_acceptance.py:277-297):

    pull one-shot   RX (N-1) M            (every rank reads all N-1 peer buckets)
    pull two-shot   RX 2 (N-1)/N M        (reduce-scatter reads + all-gather reads)
    push two-shot   TX 2 (N-1)/N M        (every NVLink byte is a store)
    push one-shot   TX (N-1) M
    LL              TX 2 (N-1) M          (8-byte epoch + payload words)

    torchrun --nproc-per-node N scripts/nvlink_bytes.py [--mib 64] [--reps 100]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


COUNTERS = {
    # name: (TX field, RX field, unit bytes)
    "count_bytes": (202, 204, 1),  # NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / RCV_BYTES (Blackwell)
    "throughput_data_kib": (138, 139, 1024),  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / RX
    "throughput_raw_kib": (140, 141, 1024),  # NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX / RX
}


def nvlink_counters(handle, pynvml):
    """{counter: (TX bytes, RX bytes, links answering)} summed over this GPU's NVLinks."""
    out = {}
    for name, (ftx, frx, unit) in COUNTERS.items():
        tx = rx = links = 0
        for link in range(18):
            try:
                res = pynvml.nvmlDeviceGetFieldValues(handle, [(ftx, link), (frx, link)])
            except Exception:
                continue
            if res[0].nvmlReturn == 0 and res[1].nvmlReturn == 0:
                links += 1
                tx += int(res[0].value.ullVal) * unit
                rx += int(res[1].value.ullVal) * unit
        out[name] = (tx, rx, links)
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--ll-kib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=100)
    args = ap.parse_args()
    import pynvml
    import torch

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import open_session_dist

    class A:
        gpus = int(os.environ.get("WORLD_SIZE", "1"))

    rank, world, local = bench._dist_setup(A())
    device = torch.device("cuda", local)
    pynvml.nvmlInit()
    handle = pynvml.nvmlDeviceGetHandleByIndex(local)
    m_bytes = args.mib << 20
    _, session = open_session_dist(capacity_bytes=m_bytes + (1 << 20))
    comm = session.comm
    buf = torch.ones(m_bytes // 4, device=device)
    stream = torch.cuda.Stream(device=device)
    algos = {"oneshot": (_native.ALGO_ONESHOT, m_bytes), "twoshot": (_native.ALGO_TWOSHOT, m_bytes),
             "push_twoshot": (_native.ALGO_PUSH, m_bytes), "push_oneshot": (_native.ALGO_PUSH_ONESHOT, m_bytes // 4),
             "ll": (_native.ALGO_LL, args.ll_kib << 10)}
    if world == 2:  # at N = 2 the push one-shot rows for M fit the slot too
        algos["push_oneshot"] = (_native.ALGO_PUSH_ONESHOT, m_bytes // 2)
    expected = {
        "oneshot": ("rx", lambda m: (world - 1) * m),
        "twoshot": ("rx", lambda m: 2 * (world - 1) / world * m),
        "push_twoshot": ("tx", lambda m: 2 * (world - 1) / world * m),
        "push_oneshot": ("tx", lambda m: (world - 1) * m),
        "ll": ("tx", lambda m: 2 * (world - 1) * m),
    }
    out = {"world": world, "reps": args.reps, "rank": rank, "algos": {}}
    for name, (algo, nbytes) in algos.items():
        n = nbytes // 4
        table = _native.DeviceTable([(buf.data_ptr(), n, 0)])
        sec = ctypes.c_double()
        # warm-up outside the counters
        _native.call("mgw_time_exchange", comm, table.ptr, 1, n, None, algo, 4, 3, 0, ctypes.byref(sec),
                     stream.cuda_stream)
        torch.cuda.synchronize()
        bench._barrier(world)
        time.sleep(0.2)
        before = nvlink_counters(handle, pynvml)
        _native.call("mgw_time_exchange", comm, table.ptr, 1, n, None, algo, 4, args.reps, 0, ctypes.byref(sec),
                     stream.cuda_stream)
        torch.cuda.synchronize()
        time.sleep(0.2)
        after = nvlink_counters(handle, pynvml)
        table.close()
        bench._barrier(world)
        direction, formula = expected[name]
        want = formula(nbytes)
        rec = {"bytes": nbytes, "expected_" + direction: round(want), "exchange_us": round(sec.value * 1e6, 2)}
        for cname in COUNTERS:
            tx = (after[cname][0] - before[cname][0]) / args.reps
            rx = (after[cname][1] - before[cname][1]) / args.reps
            got = tx if direction == "tx" else rx
            rec[cname] = {"tx_per_exchange": round(tx), "rx_per_exchange": round(rx), "links": after[cname][2],
                          "ratio": round(got / want, 4) if want else None}
        out["algos"][name] = rec
    session.raise_if_failed()
    session.close()
    gathered = [None] * world
    import torch.distributed as dist

    dist.all_gather_object(gathered, out)
    if rank == 0:
        print(json.dumps({"world": world, "reps": args.reps, "ranks": gathered}))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
