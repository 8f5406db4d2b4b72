"""Kernel-level measurements on one B200 (prints one JSON document).

* K1 pack / K4 unpack bandwidth vs bucket size (hold spin, CUDA events per launch)
* emulated-rank K2/K3 device time vs size (local memory; no NVLink)
* overhead of chained kernel nodes and event-record nodes inside a CUDA graph
"""

from __future__ import annotations

import ctypes
import json
import pathlib
import statistics
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1811_11141_b200 import _native  # noqa: E402


def timed(launch, reps=20, warm=3, hold_ns=5_000_000):
    s = torch.cuda.current_stream()
    _native.call("mgw_spin_ns", hold_ns, s.cuda_stream)
    marks = []
    for r in range(warm + reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        launch(s.cuda_stream)
        b.record(s)
        if r >= warm:
            marks.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) * 1e-3 for x, y in marks)


def main():
    torch.cuda.set_device(0)
    out = {"device": torch.cuda.get_device_name(0)}
    big = torch.randn((102_015_648 // 4) + 1024, device="cuda")
    bucket = torch.empty_like(big)
    rows = []
    for nbytes in [1 << k for k in range(12, 27, 2)] + [102_015_648]:
        n = nbytes // 4
        t = _native.DeviceTable([(big.data_ptr(), n, 0)])
        tp = timed(lambda h: _native.call("mgw_pack", t.ptr, 1, bucket.data_ptr(), n, ctypes.c_float(1.0), h))
        tu = timed(lambda h: _native.call("mgw_unpack", t.ptr, 1, bucket.data_ptr(), n, h))
        tc = timed(lambda h: bucket[:n].copy_(big[:n]))
        rows.append({"bytes": nbytes, "pack_us": round(tp * 1e6, 2), "pack_gbs": round(2 * nbytes / tp / 1e9, 1),
                     "unpack_us": round(tu * 1e6, 2), "unpack_gbs": round(2 * nbytes / tu / 1e9, 1),
                     "torch_copy_us": round(tc * 1e6, 2)})
        t.close()
    out["pack_unpack"] = rows

    # many small layers (BERT-like bucket): descriptor walk cost
    counts = [768] * 120 + [589824] * 4
    tensors = [torch.randn(p, device="cuda") for p in counts]
    off, trows = 0, []
    for x, p in zip(tensors, counts):
        trows.append((x.data_ptr(), p, off))
        off += p
    t = _native.DeviceTable(trows)
    tp = timed(lambda h: _native.call("mgw_pack", t.ptr, t.n, bucket.data_ptr(), off, ctypes.c_float(1.0), h))
    out["pack_124_rows"] = {"bytes": 4 * off, "us": round(tp * 1e6, 2), "gbs": round(8 * off / tp / 1e9, 1)}
    t.close()

    # emulated all-reduce device time (all ranks' buffers local): compute-side cost
    ar = []
    for world in (2, 8):
        for nbytes in (1 << 12, 1 << 20, 1 << 24):
            n = nbytes // 4
            ins = [torch.randn(n, device="cuda") for _ in range(world)]
            outs = [torch.empty(n, device="cuda") for _ in range(world)]
            ip = (ctypes.c_void_p * world)(*[x.data_ptr() for x in ins])
            op = (ctypes.c_void_p * world)(*[x.data_ptr() for x in outs])
            for algo, name in ((_native.ALGO_ONESHOT, "oneshot"), (_native.ALGO_TWOSHOT, "twoshot")):
                tt = timed(lambda h: _native.call("mgw_allreduce_emulated", ip, op, world, n, algo, h), reps=10)
                ar.append({"world": world, "bytes": nbytes, "algo": name, "all_ranks_us": round(tt * 1e6, 2)})
    out["emulated_allreduce"] = ar

    # graph overhead: 54 chained tiny packs, with / without event records between
    small = torch.randn(1024, device="cuda")
    sb = torch.empty(1024, device="cuda")
    t = _native.DeviceTable([(small.data_ptr(), 1024, 0)])
    s = torch.cuda.Stream()
    res = {}
    for with_events in (False, True):
        try:
            torch.cuda.Event(enable_timing=True, external=True)
        except TypeError:
            if with_events:
                continue
        g = torch.cuda.CUDAGraph()
        evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(108)] if with_events else []
        with torch.cuda.graph(g, stream=s):
            h = torch.cuda.current_stream().cuda_stream
            for k in range(54):
                if with_events:
                    evs[2 * k].record()
                _native.call("mgw_pack", t.ptr, 1, sb.data_ptr(), 1024, ctypes.c_float(1.0), h)
                if with_events:
                    evs[2 * k + 1].record()
        tt = timed(lambda h: g.replay(), reps=20)
        res["with_events" if with_events else "plain"] = round(tt * 1e6 / 54, 3)
    out["graph_us_per_pack_node"] = res
    t.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
