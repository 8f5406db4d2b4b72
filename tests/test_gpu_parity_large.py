"""Bit-exact parity at the BASELINE bucket sizes, on one B200.

Random fp32 (and bf16) gradients -- normal values spread over seven decades, so every
fold order gives different bits -- at the sizes the benchmarks actually move:

* ResNet-50 SyncEASGD bucket: all 54 layers of ``resnet50_like`` in one group
  (25,503,912 elements = 102 MB; 54 rows > the 40 inline rows, so the device-table path);
* VGG-16 fc6 alone (102,764,544 elements = 411 MB), the two-shot regime;
* BERT-base as one group (199 rows, 109,482,240 elements), every row misaligned;
* 16 MiB and 64 MiB single-row buckets; the LL ceiling of each N;
* every ResNet-50 per-layer (WFBP) bucket under AUTO.

Every algorithm the AUTO rule can reach at a size (and the forced alternatives) runs
through the emulated-rank entry points (``mgw_allreduce_fused[_bf16]_emulated``: each
rank's launch runs the kernel's *own* pack -- fused_pack_range / fused_pack_parts /
push pack -- then the fold phases), for N in {2, 4, 8}, and is compared bit for bit with
the oracle ring (reference fold order, allreduce_net.py:370-411; C oracle, one thread per
simulated rank).  The ResNet-50 bucket also runs with the real barrier protocol in an
in-process rank group (LocalGroup).
"""

from __future__ import annotations

import ctypes
import zlib

import numpy as np
import pytest

from oracle import ring_oracle
from paper_1811_11141_b200 import _native, bert_base_like, resnet50_like
from paper_1811_11141_b200.model_profile import vgg16_like

pytestmark = pytest.mark.gpu

A = _native
F32_ALGOS = {"ll": A.ALGO_LL, "oneshot": A.ALGO_ONESHOT, "twoshot": A.ALGO_TWOSHOT,
             "push_oneshot": A.ALGO_PUSH_ONESHOT, "push": A.ALGO_PUSH, "push_pipe": A.ALGO_PUSH_PIPE,
             "ll128": A.ALGO_LL128, "ll128_one": A.ALGO_LL128_ONESHOT}
B16_ALGOS = {"ll": A.ALGO_LL, "oneshot": A.ALGO_ONESHOT, "twoshot": A.ALGO_TWOSHOT, "push": A.ALGO_PUSH,
             "ll128": A.ALGO_LL128, "ll128_one": A.ALGO_LL128_ONESHOT}
LL_ELEMS = 262_144


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    return torch


def _ll_ceiling(n_ranks):
    return ((1 << 20) if n_ranks == 2 else ((512 << 10) if n_ranks <= 4 else (256 << 10))) // 4


def layout(case, n_ranks):
    """(row counts in bucket order -- layer high first --, element shift of every row)."""
    if case == "r50_bucket":
        return list(reversed(resnet50_like().param_counts())), 0
    if case == "vgg_fc6":
        counts = vgg16_like().param_counts()
        return [max(counts)], 0
    if case == "bert_group":
        return [p for p in reversed(bert_base_like().param_counts()) if p], 1
    if case == "mib16":
        return [4 << 20], 0
    if case == "mib64":
        return [16 << 20], 0
    if case == "ll_ceiling":
        return [_ll_ceiling(n_ranks) - 5, 5], 0
    raise KeyError(case)


class Case:
    """Per-rank pristine buckets on the device, the layer tensors the exchange works on
    (views into one flat buffer per rank, optionally misaligned), and the oracle result."""

    def __init__(self, torch, case, n_ranks, bf16):
        self.torch = torch
        counts, shift = layout(case, n_ranks)
        self.counts, self.total = counts, sum(counts)
        dtype = torch.bfloat16 if bf16 else torch.float32
        gen = torch.Generator(device="cuda").manual_seed(zlib.crc32(f"{case}-{n_ranks}-{bf16}".encode()))
        self.pristine, self.work, self.tensors = [], [], []
        host = []
        for _ in range(n_ranks):
            x = torch.randn(self.total, generator=gen, device="cuda")
            x *= torch.pow(10.0, torch.randint(-3, 4, (self.total,), generator=gen, device="cuda").float())
            x = x.to(dtype)
            self.pristine.append(x)
            host.append(x.view(torch.int16).cpu().numpy().view(np.uint16) if bf16 else x.cpu().numpy())
            flat = torch.empty(self.total + shift * len(counts) + 8, dtype=dtype, device="cuda")
            views, off = [], 0
            for p in counts:
                off += shift
                views.append(flat[off:off + p])
                off += p
            self.work.append(flat)
            self.tensors.append(views)
        if bf16:
            want = ring_oracle.ring_allreduce_bf16(host)
            self.want = torch.from_numpy(want.view(np.int16)).cuda()
        else:
            want = ring_oracle.ring_allreduce(host)[0]
            self.want = torch.from_numpy(want.view(np.int32)).cuda()
        del host
        self.bf16 = bf16

    def reset(self):
        for r, views in enumerate(self.tensors):
            off = 0
            for t, p in zip(views, self.counts):
                t.copy_(self.pristine[r][off:off + p])
                off += p

    def run_emulated(self, algo):
        torch = self.torch
        self.reset()
        n_ranks = len(self.tensors)
        tables, slots = [], []
        dtype = torch.bfloat16 if self.bf16 else torch.float32
        for views in self.tensors:
            rows, off = [], 0
            for t, p in zip(views, self.counts):
                rows.append((t.data_ptr(), p, off))
                off += p
            tables.append(_native.DeviceTable(rows))
            slots.append(torch.empty(self.total, dtype=dtype, device="cuda"))
        tp = (ctypes.c_void_p * n_ranks)(*[t.ptr for t in tables])
        sp = (ctypes.c_void_p * n_ranks)(*[x.data_ptr() for x in slots])
        fn = "mgw_allreduce_fused_bf16_emulated" if self.bf16 else "mgw_allreduce_fused_emulated"
        _native.call(fn, tp, sp, n_ranks, self.total, ctypes.c_float(1.0), algo,
                     torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        for t in tables:
            t.close()
        del slots

    def mismatches(self):
        torch = self.torch
        bad = []
        for r, views in enumerate(self.tensors):
            got = torch.cat([v.reshape(-1) for v in views]).view(torch.int16 if self.bf16 else torch.int32)
            n_bad = int((got != self.want).sum())
            if n_bad:
                bad.append((r, n_bad, int((got != self.want).nonzero()[0])))
        return bad


_cache: dict = {}


def get_case(torch, case, n_ranks, bf16=False):
    key = (case, n_ranks, bf16)
    if key not in _cache:
        _cache.clear()  # one big case resident at a time
        torch.cuda.empty_cache()
        _cache[key] = Case(torch, case, n_ranks, bf16)
    return _cache[key]


def f32_algos(case, n_ranks):
    counts, _ = layout(case, n_ranks)
    n = sum(counts)
    out = ["oneshot", "twoshot", "push", "push_pipe", "ll128"]
    if n <= LL_ELEMS:
        out.append("ll")
    if 4 * n <= (16 << 20):
        out.extend(["push_oneshot", "ll128_one"])
    return out


F32_CASES = [(c, n, a) for c in ("ll_ceiling", "mib16", "mib64", "r50_bucket", "bert_group", "vgg_fc6")
             for n in (2, 4, 8) for a in f32_algos(c, n)]


@pytest.mark.parametrize("case,n_ranks,algo", F32_CASES, ids=[f"{c}-N{n}-{a}" for c, n, a in F32_CASES])
def test_fp32_bucket_bit_exact(torch_cuda, case, n_ranks, algo):
    c = get_case(torch_cuda, case, n_ranks)
    c.run_emulated(F32_ALGOS[algo])
    assert c.mismatches() == []


B16_CASES = [(c, n, a) for c in ("ll_ceiling", "mib16", "r50_bucket", "vgg_fc6") for n in (2, 4, 8)
             for a in (["oneshot", "twoshot", "push", "ll128"] + (["ll"] if sum(layout(c, n)[0]) <= 2 * LL_ELEMS else [])
                       + (["ll128_one"] if sum(layout(c, n)[0]) <= (8 << 20) else []))]


@pytest.mark.parametrize("case,n_ranks,algo", B16_CASES, ids=[f"{c}-N{n}-{a}" for c, n, a in B16_CASES])
def test_bf16_bucket_bit_exact(torch_cuda, case, n_ranks, algo):
    c = get_case(torch_cuda, case, n_ranks, bf16=True)
    c.run_emulated(B16_ALGOS[algo])
    assert c.mismatches() == []


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_r50_wfbp_layer_buckets_auto(torch_cuda, n_ranks):
    """Every ResNet-50 per-layer bucket (16 KiB .. 9 MiB), under the algorithm AUTO picks
    for it at this N (LL / push one-shot / pull one-shot / two-shot / push)."""
    from paper_1811_11141_b200.allreduce_net import _auto_rule
    from types import SimpleNamespace

    torch = torch_cuda
    sess = SimpleNamespace(config=SimpleNamespace(n_workers=n_ranks))
    counts = resnet50_like().param_counts()
    gen = torch.Generator(device="cuda").manual_seed(n_ranks)
    for layer, p in enumerate(counts, start=1):
        algo = _auto_rule(sess, p, fused=True)
        ins = [torch.randn(p, generator=gen, device="cuda") for _ in range(n_ranks)]
        want = ring_oracle.ring_allreduce([x.cpu().numpy() for x in ins])[0]
        tables = [_native.DeviceTable([(x.data_ptr(), p, 0)]) for x in ins]
        slots = [torch.empty(p, device="cuda") for _ in range(n_ranks)]
        tp = (ctypes.c_void_p * n_ranks)(*[t.ptr for t in tables])
        sp = (ctypes.c_void_p * n_ranks)(*[x.data_ptr() for x in slots])
        _native.call("mgw_allreduce_fused_emulated", tp, sp, n_ranks, p, ctypes.c_float(1.0), algo,
                     torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        for t in tables:
            t.close()
        for r, x in enumerate(ins):
            assert np.array_equal(x.cpu().numpy().view("<u4"), want.view("<u4")), (layer, p, algo, r)


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_r50_bucket_real_barriers_auto(torch_cuda, n_ranks):
    """The 102 MB SyncEASGD bucket (54 rows) under AUTO (push two-shot) with the real flag
    barriers: every rank's CTAs in one cooperative launch (in-process rank group)."""
    from paper_1811_11141_b200.allreduce_net import LocalGroup

    torch = torch_cuda
    c = get_case(torch, "r50_bucket", n_ranks)
    c.reset()
    torch.cuda.synchronize()
    with LocalGroup(n_ranks, device=0, capacity_bytes=4 * c.total, timeout=20.0) as grp:
        assert grp.allreduce_fused(c.tensors) == [None] * n_ranks
    assert c.mismatches() == []
