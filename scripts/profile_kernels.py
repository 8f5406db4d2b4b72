"""Single-GPU kernel workload for ncu (--set full): the hot kernels at bench sizes.

  K1 pack / K4 unpack   whole ResNet-50 bucket (102,015,648 B, 54 layers, SyncEASGD group)
  K1 pack               BERT-base-like group: 120 tensors of 768 + 4 of 589,824 (row walk)
  K2 one-shot           4 emulated ranks x 1 MiB   (local memory: same code as the IPC path
  K3 two-shot           4 emulated ranks x 64 MiB   minus the barriers and NVLink)
  fused two-shot        4 emulated ranks, ResNet-50 layer table
  fused N=1             the single-rank group kernel on the whole ResNet-50 table
  bf16 two-shot         4 emulated ranks, ResNet-50 layer table in bf16
"""

from __future__ import annotations

import ctypes
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1811_11141_b200 import _native, resnet50_like  # noqa: E402


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream().cuda_stream
    prof = resnet50_like()
    counts = list(reversed(prof.param_counts()))  # layer high first (SyncEASGD bucket)
    layers = [torch.randn(p, device="cuda") for p in counts]
    rows, off = [], 0
    for x, p in zip(layers, counts):
        rows.append((x.data_ptr(), p, off))
        off += p
    table = _native.DeviceTable(rows)
    bucket = torch.empty(off, device="cuda")
    for _ in range(2):
        _native.call("mgw_pack", table.ptr, table.n, bucket.data_ptr(), off, ctypes.c_float(1.0), s)
        _native.call("mgw_unpack", table.ptr, table.n, bucket.data_ptr(), off, s)
    bcounts = [768] * 120 + [589824] * 4
    bl = [torch.randn(p, device="cuda") for p in bcounts]
    brows, boff = [], 0
    for x, p in zip(bl, bcounts):
        brows.append((x.data_ptr(), p, boff))
        boff += p
    btable = _native.DeviceTable(brows)
    _native.call("mgw_pack", btable.ptr, btable.n, bucket.data_ptr(), boff, ctypes.c_float(1.0), s)
    world = 4
    for n_bytes, algo in ((1 << 20, _native.ALGO_ONESHOT), (64 << 20, _native.ALGO_TWOSHOT)):
        n = n_bytes // 4
        ins = [torch.randn(n, device="cuda") for _ in range(world)]
        outs = [torch.empty(n, device="cuda") for _ in range(world)]
        ip = (ctypes.c_void_p * world)(*[x.data_ptr() for x in ins])
        op = (ctypes.c_void_p * world)(*[x.data_ptr() for x in outs])
        _native.call("mgw_allreduce_emulated", ip, op, world, n, algo, s)
    tables, slots = [], []
    for r in range(world):
        ls = [torch.randn(p, device="cuda") for p in counts]
        rr, o = [], 0
        for x, p in zip(ls, counts):
            rr.append((x.data_ptr(), p, o))
            o += p
        tables.append((_native.DeviceTable(rr), ls))
        slots.append(torch.empty(o, device="cuda"))
    tp = (ctypes.c_void_p * world)(*[t.ptr for t, _ in tables])
    sp = (ctypes.c_void_p * world)(*[x.data_ptr() for x in slots])
    _native.call("mgw_allreduce_fused_emulated", tp, sp, world, off, ctypes.c_float(1.0), _native.ALGO_TWOSHOT, s)
    # single-rank fused group kernel (bench N=1 dominant kernel), whole-model table
    sec = ctypes.c_double()
    _native.call("mgw_time_exchange", None, table.ptr, table.n, off, bucket.data_ptr(), 0, 4, 1, 0,
                 ctypes.byref(sec), s)
    # bf16 gradients, fp32 accumulation: 4 emulated ranks
    btables, bslots = [], []
    for r in range(world):
        ls = [torch.randn(p, device="cuda").to(torch.bfloat16) for p in counts]
        rr, o = [], 0
        for x, p in zip(ls, counts):
            rr.append((x.data_ptr(), p, o))
            o += p
        btables.append((_native.DeviceTable(rr), ls))
        bslots.append(torch.empty(o, dtype=torch.bfloat16, device="cuda"))
    tp = (ctypes.c_void_p * world)(*[t.ptr for t, _ in btables])
    sp = (ctypes.c_void_p * world)(*[x.data_ptr() for x in bslots])
    _native.call("mgw_allreduce_fused_bf16_emulated", tp, sp, world, off, ctypes.c_float(1.0), _native.ALGO_TWOSHOT, s)
    torch.cuda.synchronize()
    print("profile workload done")


if __name__ == "__main__":
    main()
