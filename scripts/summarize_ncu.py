"""Summarise ncu outputs into profiles/: the launch list (per-kernel count, total and
share of device time) and the key metrics of a --set full capture.

    python scripts/summarize_ncu.py launches.csv prof.ncu-rep out_prefix
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def _base(name):
    """Kernel name without its parameter list, keeping template arguments
    (``rows_kernel<(mgw::RowOp)0, true>(...)`` -> ``rows_kernel<(mgw::RowOp)0, true>``)."""
    depth = 0
    for i, ch in enumerate(name):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            return name[:i]
    return name


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows:
        name = _base(r["Kernel Name"])
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    total = sum(t for _, t in agg.values())
    return {
        "launches": len(rows),
        "kernels": [
            {"kernel": k, "launches": c, "total_us": round(t, 1), "mean_us": round(t / c, 3), "share": round(t / total, 4)}
            for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])
        ],
    }


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        entry = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                entry[k] = r[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        res.append(entry)
    return res


def main():
    launch_csv, rep, prefix = sys.argv[1:4]
    doc = {"launch_list": launches(launch_csv), "full_capture": full(rep)}
    with open(prefix + ".json", "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc["launch_list"], indent=1))


if __name__ == "__main__":
    main()
