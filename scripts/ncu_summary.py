"""Summarise an `ncu --set full` report: per kernel, the mean over captured launches of
duration, DRAM bytes read / written, DRAM throughput, grid, registers and the top stall
reasons; stamped with the git HEAD the report was taken at.

    python scripts/ncu_summary.py REPORT.ncu-rep OUT.json [--sha SHA] [--note TEXT]
        [--traffic "KEY=kernel-regex" ...]     # merge mean dram read+write bytes per launch
                                               # into profiles/roofline_traffic.json as KEY
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg_throttle",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def kernel_base(name: str) -> str:
    depth = 0
    for i, ch in enumerate(name):
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0:
            return name[:i]
    return name


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--sha", default=None)
    ap.add_argument("--note", default="")
    ap.add_argument("--traffic", action="append", default=[])
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    name_col = hdr.index("Kernel Name")
    per = collections.defaultdict(list)
    for r in rows[2:]:
        rec = {"name": r[name_col]}
        for m, short in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    rec[short] = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        per[kernel_base(r[name_col])].append(rec)
    kernels = {}
    for k, recs in per.items():
        agg = {"launches": len(recs)}
        for short in METRICS.values():
            vals = [x[short] for x in recs if short in x]
            if vals:
                agg[short] = round(sum(vals) / len(vals), 3)
        if "dram_read_bytes" in agg:
            agg["dram_bytes_per_launch"] = round(agg["dram_read_bytes"] + agg.get("dram_write_bytes", 0.0))
        kernels[k] = agg
    sha = args.sha or subprocess.run(["git", "-C", str(ROOT), "rev-parse", "--short=12", "HEAD"],
                                     capture_output=True, text=True).stdout.strip()
    doc = {"report": pathlib.Path(args.report).name, "sha": sha, "note": args.note,
           "units": "duration us, bytes, pct of peak", "kernels": kernels}
    pathlib.Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")
    if args.traffic:
        tpath = ROOT / "profiles" / "roofline_traffic.json"
        traffic = json.loads(tpath.read_text()) if tpath.exists() else {}
        for spec in args.traffic:
            key, pat = spec.rsplit("=", 1)  # keys may hold "=" (e.g. "(N=1)"), kernel regexes do not
            hits = [v for k, v in kernels.items() if re.search(pat, k)]
            if hits:
                traffic[key] = hits[0]["dram_bytes_per_launch"]
                traffic.setdefault("_sources", {})[key] = {"report": doc["report"], "sha": sha}
        tpath.write_text(json.dumps(traffic, indent=1) + "\n")
    print(json.dumps({k: {kk: v[kk] for kk in ("launches", "duration_us", "dram_bytes_per_launch", "dram_throughput_pct")
                          if kk in v} for k, v in kernels.items()}, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
