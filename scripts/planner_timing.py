"""Planner (Algorithm 1) and simulator timing, this package vs the unmodified reference
(imported from /root/reference when present), on the SURVEY §8 profiles.  CPU only.

    python scripts/planner_timing.py > profiles/planner_timing_r01.json
"""

from __future__ import annotations

import importlib
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = pathlib.Path("/root/reference/pkg/src")


def best_of(fn, reps=5):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    import paper_1811_11141_b200 as ours

    ref = None
    if REF.exists():
        sys.path.insert(0, str(REF))
        ref = importlib.import_module("mgwfbp")
    models = {"nvlink_fit": (1.6e-5, 2.9e-12), "merge_heavy": (5e-3, 2.9e-12)}
    cases = {
        "resnet50_like": lambda m: m.resnet50_like(),
        "googlenet_like": lambda m: m.googlenet_like(),
        "synth_1000": lambda m: m.synth_profile(1000, param_range=(1024, 16_777_216), seed=0),
    }
    rows = []
    for (mname, model), (name, make) in [(mm, c) for mm in models.items() for c in cases.items()]:
        row = {"profile": name, "model": mname}
        for tag, m in (("ours", ours), ("reference", ref)):
            if m is None:
                continue
            prof = make(m)
            cm = m.CommModel(*model)
            plan = m.find_merge_plan(prof, cm)
            row[f"{tag}_plan_ms"] = round(best_of(lambda: m.find_merge_plan(prof, cm)) * 1e3, 3)
            row[f"{tag}_simulate_ms"] = round(best_of(lambda: m.simulate_mgwfbp(prof, cm, plan)) * 1e3, 3)
            row[f"{tag}_merged"] = sorted(plan.merged_layers)
            row["groups"] = len(plan.groups())
        if ref is not None:
            row["identical_plans"] = row["ours_merged"] == row["reference_merged"]
        row.pop("ours_merged", None)
        row.pop("reference_merged", None)
        row["layers"] = make(ours).num_layers
        rows.append(row)
    print(json.dumps({"models": models, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
