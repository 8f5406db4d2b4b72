"""Pair an ncu --set full capture of the bench's N=1 step (scripts/profile_step.py) with
the per-group algorithmic bytes: DRAM traffic per launch of the dominant kernel (the
fused N=1 group kernel) vs algorithmic bytes.

    python scripts/summarize_step.py step.ncu-rep profile_step_groups.json out.json

Writes the summary and merges ``"<kernel>@N1"`` (mean dram read+write bytes per launch)
into profiles/roofline_traffic.json, which bench.py reports as ``roofline.traffic``.
"""

from __future__ import annotations

import csv
import io
import json
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _num(v):
    return float(v.replace(",", "")) if v not in ("", "n/a") else 0.0


def main():
    rep, groups_path, out_path = sys.argv[1:4]
    traffic_path = pathlib.Path(sys.argv[4]) if len(sys.argv) > 4 else ROOT / "profiles" / "roofline_traffic.json"
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {k: hdr.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                     "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                                     "launch__grid_size")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    launches = []
    for r in rows[2:]:
        if "fused_oneshot_kernel" not in r[col["Kernel Name"]]:
            continue
        get = lambda k: _num(r[col[k]]) * scale.get(units[col[k]], 1)  # noqa: E731
        launches.append({"us": get("gpu__time_duration.sum") * 1e6,
                         "dram_bytes": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
                         "dram_pct": _num(r[col["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]]),
                         "grid": int(_num(r[col["launch__grid_size"]]))})
    meta = json.loads(pathlib.Path(groups_path).read_text())
    alg = meta["algorithmic_bytes"]
    n = min(len(alg), len(launches))
    if n == 0:
        raise SystemExit("no fused N=1 launches in the capture")
    launches, alg = launches[:n], alg[:n]
    mean_traffic = sum(l["dram_bytes"] for l in launches) / n
    mean_alg = sum(alg) / n
    summary = {
        "what": "ncu --set full --clock-control none of the bench's N=1 MG-WFBP step (scripts/profile_step.py), "
                "fused N=1 group kernel launches in send order; ncu serialises and cold-starts every launch",
        "launches": n,
        "mean_algorithmic_bytes": round(mean_alg),
        "mean_dram_bytes": round(mean_traffic),
        "traffic_over_algorithmic": round(mean_traffic / mean_alg, 4),
        "sum_us": round(sum(l["us"] for l in launches), 2),
        "per_launch": [dict(l, algorithmic_bytes=a) for l, a in zip(launches, alg)],
    }
    pathlib.Path(out_path).write_text(json.dumps(summary, indent=1))
    tf = traffic_path
    merged = json.loads(tf.read_text()) if tf.exists() else {}
    merged[f"{meta['kernel']}@N1"] = round(mean_traffic)
    merged["_note"] = ("mean dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel "
                       "from one ncu --set full capture (scripts/summarize_step.py); multi-rank kernels "
                       "cannot be replayed by ncu, so N>1 stays null")
    tf.write_text(json.dumps(merged, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k != "per_launch"}))


if __name__ == "__main__":
    main()
