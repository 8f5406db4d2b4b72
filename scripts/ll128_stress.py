"""Long randomized stress of the LL128 kernels over real IPC ranks (one process per GPU):
`iterations` back-to-back collectives per rank, random sizes / row splits / dtypes, only
the LL128 one-shot and two-shot, iteration-dependent exact payloads (a stale 128-B line can
never pass for fresh data).  Prints one JSON line: failures per rank.

    python scripts/ll128_stress.py --ranks 4 --iterations 1500
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys
import time
from functools import partial

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--iterations", type=int, default=1500)
    ap.add_argument("--max-elems", type=int, default=1 << 23)
    ap.add_argument("--seed", type=int, default=7)
    args = ap.parse_args()
    import _mp_tasks

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import run_workers

    only = (_native.ALGO_LL128, _native.ALGO_LL128_ONESHOT)
    t0 = time.time()
    res = run_workers(args.ranks, partial(_mp_tasks.stress_task, iterations=args.iterations, seed=args.seed,
                                          only=only, max_n=args.max_elems),
                      timeout=3000, capacity_bytes=(args.max_elems * 4 * 9) // 8 * args.ranks + (1 << 20))
    out = {"ranks": args.ranks, "iterations": args.iterations, "max_elems": args.max_elems,
           "algorithms": ["ll128_twoshot", "ll128_oneshot"], "wall_s": round(time.time() - t0, 1),
           "failures": {str(r): v[0] for r, v in res.items()}, "first": {str(r): v[1] for r, v in res.items()}}
    print(json.dumps(out))
    return 0 if all(v[0] == 0 for v in res.values()) else 1


if __name__ == "__main__":
    raise SystemExit(main())
