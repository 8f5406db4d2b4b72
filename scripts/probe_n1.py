"""Self-timed phases of the single-rank group kernel (pack -> one-input fold -> write-back)
at several group sizes: where a small group's ~2 us in-step span goes.

    python scripts/probe_n1.py
"""

from __future__ import annotations

import ctypes
import json
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main() -> int:
    import torch

    from paper_1811_11141_b200 import _native

    torch.cuda.set_device(0)
    comm = ctypes.c_void_p()
    _native.call("mgw_comm_create", 0, 1, 0, 64 << 20, ctypes.byref(comm), None)
    out = {}
    for nbytes in (16384, 65536, 262144, 1 << 20, 4 << 20, 9437184):
        n = nbytes // 4
        x = torch.randn(n, device="cuda")
        table = _native.DeviceTable([(x.data_ptr(), n, 0)])
        reps = 40
        buf = (ctypes.c_uint64 * (reps * 8))()
        _native.call("mgw_probe_phases", comm, table.ptr, 1, n, 0, reps, buf, torch.cuda.current_stream().cuda_stream)
        rows = [list(buf[r * 8:(r + 1) * 8]) for r in range(5, reps)]

        def med(f):
            return round(statistics.median(f(r) for r in rows) / 1e3, 3)

        out[nbytes] = {
            "span_us": med(lambda r: r[1] - r[0]),
            "cta0_entry_after_first_us": med(lambda r: r[2] - r[0]),
            "cta0_pack_us": med(lambda r: r[3] - r[2]),
            "cta0_fold_writeback_us": med(lambda r: r[5] - r[4]),
            "cta0_done_to_last_exit_us": med(lambda r: r[1] - r[5]),
        }
        table.close()
    _native.lib().mgw_comm_destroy(comm)
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
