"""Per-group kernel spans of the bench's N=1 MG-WFBP iteration (B200 ResNet-50 profile,
CUDA graph, fused group kernel): where the in-step time of the dominant kernel goes.

    python scripts/group_spans.py [--iters 10]
"""

from __future__ import annotations

import argparse
import json
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--local-min-slots", type=int, default=0)
    args = ap.parse_args()
    import torch

    from paper_1811_11141_b200 import MergePlan, _native
    from paper_1811_11141_b200.overlap import OverlappedIteration

    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    if args.local_min_slots:
        _native.call("mgw_set_option", _native.OPT_LOCAL_MIN_SLOTS, args.local_min_slots)
    profile, _, _ = bench.b200_profile()
    plan = MergePlan(frozenset(), profile.num_layers)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, device=device)
    it = OverlappedIteration(profile, plan, comm=None, rank=0, world=1, device=device, graph=True, fused=True,
                            pdl=not args.no_pdl)
    spans = []
    try:
        for i in range(3 + args.iters):
            with torch.cuda.stream(it.compute_stream):
                bench.l2_flush(flush)
            it.run()
            if i >= 3:
                spans.append(it.kernel_times()[1])
        ok = it.verify()
        gbytes = it.group_bytes()
    finally:
        it.close()
    rows = []
    for g, b in enumerate(gbytes):
        us = statistics.median(s[g] for s in spans) * 1e6
        rows.append({"group": g, "bytes": b, "span_us": round(us, 3),
                     "gbs_4x": round(4 * b / (us * 1e-6) / 1e9, 1) if us > 0 else None})
    total_us = sum(r["span_us"] for r in rows)
    out = {"verified": ok, "groups": len(rows), "sum_span_us": round(total_us, 2),
           "achieved_4x_gbs": round(4 * sum(gbytes) / (total_us * 1e-6) / 1e9, 1), "rows": rows}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
