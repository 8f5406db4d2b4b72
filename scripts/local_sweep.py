"""Single-rank fused group kernel (bench N=1 dominant kernel): graph-replayed step time vs
bucket size, for the library named by MGWFBP_B200_LIB (A/B of build variants)."""

from __future__ import annotations

import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    import torch

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    sizes = [65536, 262144, 1 << 20, 2 << 20, 4 << 20, 8 << 20, 9437184, 32 << 20, 102015648 // 4 * 4]
    t = bench._exchange_times(None, 1, dev, sizes, kind=4 | 256, repeats=50)
    out = {"lib": os.environ.get("MGWFBP_B200_LIB", "default"), "sizes": sizes,
           "us": [round(x * 1e6, 2) for x in t], "hbm_gbs": [round(4 * s / x / 1e9, 1) for s, x in zip(sizes, t)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
