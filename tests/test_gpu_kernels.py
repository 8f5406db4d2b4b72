"""K1 pack+scale, K4 unpack, fill/check, K5 spin, and the K2/K3 fold order -- on one B200.

Multi-rank all-reduce on one device uses the emulated-rank entry point (one launch
per rank and phase, no barriers, the same device reduction code), which is how the
fold order is checked bit-exactly against the reference's ring outputs without
running mutually-waiting kernels on one GPU."""

import ctypes

import numpy as np
import pytest

from conftest import golden_ring
from oracle import ring_oracle
from paper_1811_11141_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    return torch


def _rows_for(tensors, counts):
    rows, off = [], 0
    for t, p in zip(tensors, counts):
        rows.append((t.data_ptr(), p, off))
        off += p
    return rows, off


@pytest.mark.parametrize("counts,shift", [
    ([4096, 2359296, 1000, 3, 0 + 17, 9408], 0),   # resnet-ish + odd sizes
    ([1, 2, 3, 5, 7, 11, 13, 1 << 16], 1),         # misaligned tensor starts
    ([768] * 40 + [3072, 23440896 // 64], 3),      # many small BERT-like tensors
])
def test_pack_unpack_bitwise(torch_cuda, counts, shift):
    torch = torch_cuda
    gen = torch.Generator(device="cuda").manual_seed(7)
    bases = [torch.randn(p + shift, generator=gen, device="cuda") for p in counts]
    tensors = [b[shift:] for b in bases]
    rows, total = _rows_for(tensors, counts)
    table = _native.DeviceTable(rows)
    bucket = torch.full((total,), float("nan"), device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    _native.call("mgw_pack", table.ptr, table.n, bucket.data_ptr(), total, ctypes.c_float(1.0), stream)
    want = ring_oracle.pack_group({k + 1: t.cpu().numpy() for k, t in enumerate(reversed(tensors))},
                                  list(reversed(counts)), 1, len(counts))
    assert np.array_equal(bucket.cpu().numpy().view("<u4"), want.view("<u4"))
    outs = [torch.zeros(p + shift, device="cuda")[shift:] for p in counts]
    out_rows, _ = _rows_for(outs, counts)
    out_table = _native.DeviceTable(out_rows)
    _native.call("mgw_unpack", out_table.ptr, out_table.n, bucket.data_ptr(), total, stream)
    for a, b in zip(outs, tensors):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    table.close()
    out_table.close()


def test_pack_scale_is_exact_power_of_two(torch_cuda):
    torch = torch_cuda
    x = torch.randn(100003, device="cuda")
    table = _native.DeviceTable([(x.data_ptr(), x.numel(), 0)])
    bucket = torch.empty_like(x)
    _native.call("mgw_pack", table.ptr, 1, bucket.data_ptr(), x.numel(), ctypes.c_float(0.125),
                 torch.cuda.current_stream().cuda_stream)
    want = x.cpu().numpy() * np.float32(0.125)
    assert np.array_equal(bucket.cpu().numpy().view("<u4"), want.view("<u4"))
    table.close()


def test_fill_and_check(torch_cuda):
    torch = torch_cuda
    counts = [5, 4096, 33, 1 << 20]
    tensors = [torch.zeros(p, device="cuda") for p in counts]
    rows, _ = _rows_for(tensors, counts)
    table = _native.DeviceTable(rows)
    vals = torch.tensor([1.0, 2.0, 3.0, 4.0], device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _native.call("mgw_fill_const", table.ptr, table.n, vals.data_ptr(), s)
    for t, v in zip(tensors, (1.0, 2.0, 3.0, 4.0)):
        assert bool((t == v).all())
    bad = ctypes.c_int64()
    _native.call("mgw_check_const", table.ptr, table.n, vals.data_ptr(), ctypes.byref(bad), s)
    assert bad.value == 0
    tensors[3][17] = 0.5
    tensors[0][4] = 9.0
    _native.call("mgw_check_const", table.ptr, table.n, vals.data_ptr(), ctypes.byref(bad), s)
    assert bad.value == 2
    table.close()


def test_spin_ns_duration(torch_cuda):
    torch = torch_cuda
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _native.call("mgw_spin_ns", 100_000, s.cuda_stream)
    a.record(s)
    _native.call("mgw_spin_ns", 2_000_000, s.cuda_stream)
    b.record(s)
    b.synchronize()
    ms = a.elapsed_time(b)
    assert 1.99 <= ms < 2.3


def _emulated(torch, ins, algo, in_place=False):
    n = ins[0].numel()
    world = len(ins)
    outs = list(ins) if in_place else [torch.full((max(n, 1),), float("nan"), device="cuda")[:n] for _ in ins]
    ip = (ctypes.c_void_p * world)(*[t.data_ptr() for t in ins])
    op = (ctypes.c_void_p * world)(*[t.data_ptr() for t in outs])
    _native.call("mgw_allreduce_emulated", ip, op, world, n, algo, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("algo", [_native.ALGO_ONESHOT, _native.ALGO_TWOSHOT])
@pytest.mark.parametrize("n_ranks", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 17, 1001, 4099])
def test_fold_order_bit_exact_vs_reference_ring(torch_cuda, algo, n_ranks, n):
    torch = torch_cuda
    g = golden_ring()
    ins = [torch.from_numpy(g[f"in_N{n_ranks}_n{n}_r{r}"].copy()).cuda() for r in range(n_ranks)]
    want = g[f"out_N{n_ranks}_n{n}"]
    for out in _emulated(torch, ins, algo):
        assert np.array_equal(out.cpu().numpy().view("<u4"), want.view("<u4"))


@pytest.mark.parametrize("algo", [_native.ALGO_ONESHOT, _native.ALGO_TWOSHOT])
@pytest.mark.parametrize("n_ranks", [2, 5, 7, 8])
def test_fold_order_large_vs_oracle(torch_cuda, algo, n_ranks):
    torch = torch_cuda
    n = (1 << 20) + 3
    rng = np.random.default_rng(n_ranks)
    host = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)).astype("<f4") for _ in range(n_ranks)]
    want = ring_oracle.ring_allreduce(host)[0]
    ins = [torch.from_numpy(h.copy()).cuda() for h in host]
    for out in _emulated(torch, ins, algo):
        assert np.array_equal(out.cpu().numpy().view("<u4"), want.view("<u4"))


def test_twoshot_in_place(torch_cuda):
    torch = torch_cuda
    n = 12345
    host = [np.random.default_rng(r).standard_normal(n).astype("<f4") for r in range(4)]
    want = ring_oracle.ring_allreduce(host)[0]
    ins = [torch.from_numpy(h.copy()).cuda() for h in host]
    for out in _emulated(torch, ins, _native.ALGO_TWOSHOT, in_place=True):
        assert np.array_equal(out.cpu().numpy().view("<u4"), want.view("<u4"))


def test_integer_payloads_exact(torch_cuda):
    """The reference's exact-sum payloads (allreduce_net tests): arange + rank, rank + 1."""
    torch = torch_cuda
    for world in (2, 3, 4, 8):
        ins = [torch.arange(23, dtype=torch.float32, device="cuda") + r for r in range(world)]
        want = torch.arange(23, dtype=torch.float32, device="cuda") * world + world * (world - 1) / 2
        for algo in (_native.ALGO_ONESHOT, _native.ALGO_TWOSHOT):
            for out in _emulated(torch, ins, algo):
                assert torch.equal(out, want)
        ones = [torch.full((1_000_000,), float(r + 1), device="cuda") for r in range(world)]
        for out in _emulated(torch, ones, _native.ALGO_TWOSHOT):
            assert bool((out == world * (world + 1) / 2).all())


def _fused_emulated(torch, per_rank_tensors, counts, algo, scale=1.0):
    """Emulated fused kernel: every rank packs its own layer tensors, folds, writes back."""
    world = len(per_rank_tensors)
    tables, slots = [], []
    total = sum(counts)
    for tensors in per_rank_tensors:
        rows, off = [], 0
        for x, p in zip(tensors, counts):
            rows.append((x.data_ptr(), p, off))
            off += p
        tables.append(_native.DeviceTable(rows))
        slots.append(torch.full((total,), float("nan"), device="cuda"))
    tp = (ctypes.c_void_p * world)(*[t.ptr for t in tables])
    sp = (ctypes.c_void_p * world)(*[x.data_ptr() for x in slots])
    _native.call("mgw_allreduce_fused_emulated", tp, sp, world, total, ctypes.c_float(scale), algo,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for t in tables:
        t.close()


@pytest.mark.parametrize("algo", [_native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_PUSH,
                                  _native.ALGO_PUSH_ONESHOT, _native.ALGO_LL, _native.ALGO_PUSH_PIPE,
                                  _native.ALGO_LL128, _native.ALGO_LL128_ONESHOT])
@pytest.mark.parametrize("n_ranks", [2, 3, 4, 8])
@pytest.mark.parametrize("shift", [0, 1])
def test_fused_exchange_bit_exact(torch_cuda, algo, n_ranks, shift):
    """Fused pack -> fold -> write-back equals oracle pack + reference ring + unpack, bit for bit,
    for a layer mix with odd sizes, misaligned tensors and a tail."""
    torch = torch_cuda
    counts = [9408, 4096, 1001, 3, 36864, 17, 2049]  # layer high first
    rng = np.random.default_rng(100 + n_ranks)
    host = [[(rng.standard_normal(p) * 10.0 ** rng.integers(-2, 3, p)).astype("<f4") for p in counts]
            for _ in range(n_ranks)]
    tensors = []
    for r in range(n_ranks):
        ts = []
        for h in host[r]:
            base = torch.empty(h.size + shift, device="cuda")
            t = base[shift:]
            t.copy_(torch.from_numpy(h))
            ts.append(t)
        tensors.append(ts)
    _fused_emulated(torch, tensors, counts, algo)
    buckets = [np.concatenate(host[r]) for r in range(n_ranks)]
    want = ring_oracle.ring_allreduce(buckets)[0]
    off = 0
    for k, p in enumerate(counts):
        for r in range(n_ranks):
            got = tensors[r][k].cpu().numpy()
            assert np.array_equal(got.view("<u4"), want[off:off + p].view("<u4")), (r, k)
        off += p


def test_fused_exchange_many_rows_from_device_table(torch_cuda):
    """More layers than fit in the kernel parameters (BERT-like: 124 tiny + big rows)."""
    torch = torch_cuda
    counts = [768] * 60 + [3072, 589824] + [768] * 60
    n_ranks = 4
    rng = np.random.default_rng(5)
    host = [[rng.standard_normal(p).astype("<f4") for p in counts] for _ in range(n_ranks)]
    tensors = [[torch.from_numpy(h).cuda() for h in host[r]] for r in range(n_ranks)]
    _fused_emulated(torch, tensors, counts, _native.ALGO_TWOSHOT, scale=0.25)
    buckets = [np.concatenate(host[r]) * np.float32(0.25) for r in range(n_ranks)]
    want = ring_oracle.ring_allreduce(buckets)[0]
    got = np.concatenate([t.cpu().numpy() for t in tensors[2]])
    assert np.array_equal(got.view("<u4"), want.view("<u4"))


@pytest.mark.parametrize("algo", [_native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_LL, _native.ALGO_PUSH,
                                  _native.ALGO_LL128, _native.ALGO_LL128_ONESHOT])
@pytest.mark.parametrize("n_ranks", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("shift,scale", [(0, 1.0), (1, 1.0), (3, 0.125)])
def test_bf16_exchange_bit_exact(torch_cuda, algo, n_ranks, shift, scale):
    """bf16 gradients, fp32 accumulation: fused pack -> fold -> write-back
    equals the oracle (reference fold over upcast inputs, rounded once), bit for bit, for odd
    row sizes, misaligned tensors, segment-straddling slots and an n % 8 tail."""
    torch = torch_cuda
    if algo in (_native.ALGO_LL, _native.ALGO_PUSH, _native.ALGO_LL128, _native.ALGO_LL128_ONESHOT) and n_ranks == 1:
        pytest.skip("LL / push / LL128 need >= 2 ranks")
    counts = [9408, 4096, 1001, 3, 36864, 17, 2049, 8, 7]  # layer high first
    total = sum(counts)
    rng = np.random.default_rng(300 + n_ranks)
    host = [[ring_oracle.bf16_round((rng.standard_normal(p) * 10.0 ** rng.integers(-3, 4, p)).astype("<f4"))
             for p in counts] for _ in range(n_ranks)]
    tensors, tables, slots = [], [], []
    for r in range(n_ranks):
        ts, rows, off = [], [], 0
        for h, p in zip(host[r], counts):
            base = torch.empty(p + shift, dtype=torch.bfloat16, device="cuda")
            t = base[shift:]
            t.copy_(torch.from_numpy(h.view(np.int16)).view(torch.bfloat16))
            ts.append(t)
            rows.append((t.data_ptr(), p, off))
            off += p
        tensors.append(ts)
        tables.append(_native.DeviceTable(rows))
        slots.append(torch.full((total,), float("nan"), dtype=torch.bfloat16, device="cuda"))
    tp = (ctypes.c_void_p * n_ranks)(*[t.ptr for t in tables])
    sp = (ctypes.c_void_p * n_ranks)(*[x.data_ptr() for x in slots])
    _native.call("mgw_allreduce_fused_bf16_emulated", tp, sp, n_ranks, total, ctypes.c_float(scale), algo,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for t in tables:
        t.close()
    want = ring_oracle.ring_allreduce_bf16([np.concatenate(host[r]) for r in range(n_ranks)], scale=scale)
    off = 0
    for k, p in enumerate(counts):
        for r in range(n_ranks):
            got = tensors[r][k].view(torch.int16).cpu().numpy().view(np.uint16)
            bad = np.flatnonzero(got != want[off:off + p])
            assert bad.size == 0, (r, k, bad.size, int(bad[0]))
        off += p


def test_bf16_rejects_unsupported_algorithms(torch_cuda):
    torch = torch_cuda
    t = torch.zeros(64, dtype=torch.bfloat16, device="cuda")
    table = _native.DeviceTable([(t.data_ptr(), 64, 0)])
    tp = (ctypes.c_void_p * 2)(table.ptr, table.ptr)
    sp = (ctypes.c_void_p * 2)(t.data_ptr(), t.data_ptr())
    with pytest.raises(ValueError):
        _native.call("mgw_allreduce_fused_bf16_emulated", tp, sp, 2, 64, ctypes.c_float(1.0), _native.ALGO_NVLS,
                     torch.cuda.current_stream().cuda_stream)
    table.close()


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("misaligned_every", [0, 7])
def test_pack_unpack_paths_r50_bucket(torch_cuda, path, misaligned_every):
    """K1/K4 on the 102 MB ResNet-50 whole-model bucket through the LDG kernel (path 1) and
    the TMA bulk kernel (path 2): bitwise equal to the oracle layout (allreduce_net.py:
    499-509), with every 7th row at a misaligned tensor address (scalar fallback rows)."""
    from paper_1811_11141_b200 import resnet50_like

    torch = torch_cuda
    counts = list(reversed(resnet50_like().param_counts()))
    gen = torch.Generator(device="cuda").manual_seed(11)
    tensors = []
    for k, p in enumerate(counts):
        shift = 1 if misaligned_every and k % misaligned_every == 3 else 0
        tensors.append(torch.randn(p + shift, generator=gen, device="cuda")[shift:])
    rows, total = _rows_for(tensors, counts)
    table = _native.DeviceTable(rows)
    bucket = torch.full((total,), float("nan"), device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    try:
        _native.call("mgw_set_option", _native.OPT_ROWS_PATH, path)
        _native.call("mgw_pack", table.ptr, table.n, bucket.data_ptr(), total, ctypes.c_float(1.0), stream)
        want = torch.cat(tensors)
        assert torch.equal(bucket.view(torch.int32), want.view(torch.int32))
        outs = [torch.zeros(t.numel() + 1, device="cuda")[1 if k % 5 == 0 else 0:][:t.numel()]
                for k, t in enumerate(tensors)]
        out_rows, _ = _rows_for(outs, counts)
        out_table = _native.DeviceTable(out_rows)
        _native.call("mgw_unpack", out_table.ptr, out_table.n, bucket.data_ptr(), total, stream)
        torch.cuda.synchronize()
        for a, b in zip(outs, tensors):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32))
        out_table.close()
    finally:
        _native.call("mgw_set_option", _native.OPT_ROWS_PATH, 0)
        table.close()


@pytest.mark.parametrize("n_ranks", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [2_000_003, 4_194_304 + 1, 12_582_917])
def test_push_pipe_sub_chunks_bit_exact(torch_cuda, n_ranks, n):
    """Pipelined push two-shot with several sub-chunks per CTA chunk (sizes where S > 1),
    segment-straddling slots and an n % 4 tail: bit-exact with the reference ring."""
    torch = torch_cuda
    gen = torch.Generator(device="cuda").manual_seed(n_ranks * 31 + n)
    ins = [torch.randn(n, generator=gen, device="cuda") for _ in range(n_ranks)]
    want = ring_oracle.ring_allreduce([x.cpu().numpy() for x in ins])[0]
    tables = [_native.DeviceTable([(x.data_ptr(), n, 0)]) for x in ins]
    slots = [torch.empty(n, device="cuda") for _ in range(n_ranks)]
    tp = (ctypes.c_void_p * n_ranks)(*[t.ptr for t in tables])
    sp = (ctypes.c_void_p * n_ranks)(*[x.data_ptr() for x in slots])
    _native.call("mgw_allreduce_fused_emulated", tp, sp, n_ranks, n, ctypes.c_float(1.0), _native.ALGO_PUSH_PIPE,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for t in tables:
        t.close()
    for x in ins:
        assert np.array_equal(x.cpu().numpy().view("<u4"), want.view("<u4"))
