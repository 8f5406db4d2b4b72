"""K1 pack / K4 unpack on the ResNet-50 whole-model bucket (102 MB, 54 rows): HBM GB/s of
the LDG rows kernel vs the TMA bulk kernel (mgw_set_option(MGW_OPT_ROWS_PATH, ...)).

Each rep is timed alone with a CUDA event pair on the launching stream, after an L2 flush
(a 256 MiB write) outside the events; algorithmic bytes = 2 x bucket bytes (read + write).

    python scripts/rows_bench.py [--path 0|1|2] [--reps 20] [--out json]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--path", type=int, nargs="*", default=[1, 2])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_1811_11141_b200 import _native, resnet50_like

    torch.cuda.set_device(0)
    counts = list(reversed(resnet50_like().param_counts()))  # bucket order: layer high first
    total = sum(counts)
    flat = torch.randn(total, device="cuda")  # one contiguous gradient buffer (DDP-style)
    rows, off = [], 0
    for p in counts:
        rows.append((flat[off:off + p].data_ptr(), p, off))
        off += p
    table = _native.DeviceTable(rows)
    bucket = torch.empty(total, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    out = {"bytes": 4 * total, "rows": len(rows), "hbm_peak_gbs": hbm, "paths": {}}
    for path in args.path:
        _native.call("mgw_set_option", _native.OPT_ROWS_PATH, path)
        res = {}
        for op in ("pack", "unpack"):
            times = []
            for i in range(args.warmup + args.reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                if op == "pack":
                    _native.call("mgw_pack", table.ptr, table.n, bucket.data_ptr(), total, ctypes.c_float(1.0),
                                 s.cuda_stream)
                else:
                    _native.call("mgw_unpack", table.ptr, table.n, bucket.data_ptr(), total, s.cuda_stream)
                b.record(s)
                b.synchronize()
                if i >= args.warmup:
                    times.append(a.elapsed_time(b) * 1e-3)
            t = statistics.median(times)
            gbs = 2 * 4 * total / t / 1e9
            res[op] = {"us_median": round(t * 1e6, 2), "us_min": round(min(times) * 1e6, 2),
                       "gbs": round(gbs, 1), "frac_of_measured_hbm": round(gbs / hbm, 4)}
        # bit-exact round trip on this path
        ref = flat.clone()
        _native.call("mgw_pack", table.ptr, table.n, bucket.data_ptr(), total, ctypes.c_float(1.0), s.cuda_stream)
        flat.zero_()
        _native.call("mgw_unpack", table.ptr, table.n, bucket.data_ptr(), total, s.cuda_stream)
        torch.cuda.synchronize()
        res["round_trip_exact"] = bool(torch.equal(flat.view(torch.int32), ref.view(torch.int32)))
        flat.copy_(ref)
        out["paths"][{0: "auto", 1: "ldg", 2: "tma_bulk"}[path]] = res
    _native.call("mgw_set_option", _native.OPT_ROWS_PATH, 0)
    table.close()
    line = json.dumps(out)
    print(line)
    if args.out:
        pathlib.Path(args.out).write_text(line + "\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
