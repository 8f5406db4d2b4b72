"""The real multi-rank protocol on ONE B200: an in-process rank group (``LocalGroup``,
``mgw_comm_create_local``) whose ranks' CTAs run together in ONE cooperative launch
(``mgw_group_allreduce_fused``), so every barrier flag, LL header, push store and tag check
of the NVSwitch path executes between live, co-resident CTAs -- the driver's 1-GPU box
sees the same device code the IPC ranks run, without kernels that wait on one another
being separate launches.

Covers: every fused algorithm (fp32 LL / pull one-shot / pull two-shot / push one-shot /
push two-shot; bf16 LL / one-shot / two-shot) with the kernels' own pack, bit-exact
against the oracle ring (reference fold order, allreduce_net.py:370-411) for N in
{2, 3, 4, 8}; AUTO across its crossovers; the collective tag (the reference's frame
header check, allreduce_net.py:340-345): length, group, iteration, scale and CTA-cap
disagreements -- and two equal-size groups issued in swapped order -- raise ProtocolError
on every rank in well under a second; an absent peer times out; errors reset.
"""

from __future__ import annotations

import time

import numpy as np
import pytest

from oracle import ring_oracle
from paper_1811_11141_b200 import _native
from paper_1811_11141_b200.allreduce_net import LocalGroup, ProtocolError, group_tag

pytestmark = pytest.mark.gpu

ALGOS_F32 = [_native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_PUSH_ONESHOT,
             _native.ALGO_PUSH, _native.ALGO_PUSH_PIPE, _native.ALGO_LL128, _native.ALGO_LL128_ONESHOT]
ALGOS_B16 = [_native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_PUSH, _native.ALGO_LL128,
             _native.ALGO_LL128_ONESHOT]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    return torch


_groups: dict = {}


@pytest.fixture
def group(torch_cuda):
    """group(N) -> a cached LocalGroup (64 MB slots); closed at module end."""

    def get(n, capacity=64 << 20):
        key = (n, capacity)
        if key not in _groups:
            _groups[key] = LocalGroup(n, device=0, capacity_bytes=capacity, timeout=10.0)
        return _groups[key]

    return get


@pytest.fixture(scope="module", autouse=True)
def _close_groups():
    yield
    for g in _groups.values():
        g.close()
    _groups.clear()


def _rank_tensors(torch, host, shift, dtype):
    out = []
    for h in host:
        base = torch.empty(h.size + shift, dtype=dtype, device="cuda")
        t = base[shift:]
        if dtype == torch.bfloat16:
            t.copy_(torch.from_numpy(h.view(np.int16)).view(torch.bfloat16))
        else:
            t.copy_(torch.from_numpy(h))
        out.append(t)
    return out


def _check_f32(tensors, host, counts):
    want = ring_oracle.ring_allreduce([np.concatenate(h) for h in host])[0]
    off = 0
    for k, p in enumerate(counts):
        for r in range(len(host)):
            got = tensors[r][k].cpu().numpy()
            assert np.array_equal(got.view("<u4"), want[off:off + p].view("<u4")), (r, k)
        off += p


COUNTS = [9408, 4096, 1001, 3, 36864, 17, 2049]  # layer high first: odd sizes and a tail


@pytest.mark.parametrize("algo", ALGOS_F32)
@pytest.mark.parametrize("n_ranks", [2, 3, 4, 8])
@pytest.mark.parametrize("shift", [0, 1])
def test_fused_fp32_real_barriers_bit_exact(torch_cuda, group, algo, n_ranks, shift):
    torch = torch_cuda
    rng = np.random.default_rng(1000 + n_ranks)
    host = [[(rng.standard_normal(p) * 10.0 ** rng.integers(-2, 3, p)).astype("<f4") for p in COUNTS]
            for _ in range(n_ranks)]
    tensors = [_rank_tensors(torch, h, shift, torch.float32) for h in host]
    assert group(n_ranks).allreduce_fused(tensors, algo) == [None] * n_ranks
    _check_f32(tensors, host, COUNTS)


@pytest.mark.parametrize("algo", ALGOS_B16)
@pytest.mark.parametrize("n_ranks", [2, 4, 8])
@pytest.mark.parametrize("shift,scale", [(0, 1.0), (3, 0.125)])
def test_fused_bf16_real_barriers_bit_exact(torch_cuda, group, algo, n_ranks, shift, scale):
    torch = torch_cuda
    counts = COUNTS + [8, 7]
    rng = np.random.default_rng(2000 + n_ranks)
    host = [[ring_oracle.bf16_round((rng.standard_normal(p) * 10.0 ** rng.integers(-3, 4, p)).astype("<f4"))
             for p in counts] for _ in range(n_ranks)]
    tensors = [_rank_tensors(torch, h, shift, torch.bfloat16) for h in host]
    assert group(n_ranks).allreduce_fused(tensors, algo, scales=[scale] * n_ranks) == [None] * n_ranks
    want = ring_oracle.ring_allreduce_bf16([np.concatenate(h) for h in host], scale=scale)
    off = 0
    for k, p in enumerate(counts):
        for r in range(n_ranks):
            got = tensors[r][k].view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(got, want[off:off + p]), (r, k)
        off += p


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
@pytest.mark.parametrize("nbytes", [4096, 1 << 20, 6 << 20, 24 << 20])
def test_auto_choice_bit_exact(torch_cuda, group, n_ranks, nbytes):
    """AUTO across the LL / one-shot / two-shot / push crossovers, one tensor per rank,
    repeated so consecutive collectives alternate slot parities."""
    torch = torch_cuda
    n = nbytes // 4 + 3
    gen = torch.Generator(device="cuda").manual_seed(n_ranks * 7 + nbytes)
    for _ in range(3):
        tensors = [[torch.randn(n, generator=gen, device="cuda")] for _ in range(n_ranks)]
        host = [[t[0].cpu().numpy()] for t in tensors]
        assert group(n_ranks).allreduce_fused(tensors) == [None] * n_ranks
        _check_f32(tensors, host, [n])


def _disagree(torch, grp, n_of, *, algo=_native.ALGO_AUTO, tags=None, ctas=None, scales=None):
    """One group launch whose per-rank settings differ; returns (errors, seconds)."""
    world = grp.n_workers
    try:
        for r, sess in enumerate(grp.sessions):
            if tags is not None:
                _native.call("mgw_comm_set_group_tag", sess.comm, tags[r])
            if ctas is not None:
                _native.call("mgw_comm_set_max_ctas", sess.comm, ctas[r])
        tensors = [[torch.ones(n_of(r), device="cuda")] for r in range(world)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        errs = grp.allreduce_fused(tensors, algo, scales=scales)
        return errs, time.perf_counter() - t0
    finally:
        for sess in grp.sessions:
            _native.call("mgw_comm_set_group_tag", sess.comm, 0)
            _native.call("mgw_comm_set_max_ctas", sess.comm, 2 * 148 // world)


CASES = {
    "length": dict(n_of=lambda r: 100_000 + r),
    "length_ll": dict(n_of=lambda r: 1000 + r, algo=_native.ALGO_LL),
    "length_push": dict(n_of=lambda r: 3_000_000 + 4 * r, algo=_native.ALGO_PUSH),
    "length_pipe": dict(n_of=lambda r: 3_000_000 + 4 * r, algo=_native.ALGO_PUSH_PIPE),
    "length_ll128": dict(n_of=lambda r: 3_000_000 + 4 * r, algo=_native.ALGO_LL128),
    "length_ll128_one": dict(n_of=lambda r: 100_000 + 4 * r, algo=_native.ALGO_LL128_ONESHOT),
    "group": dict(n_of=lambda r: 100_000, tags=lambda w: [group_tag(3 + r) for r in range(w)]),
    "iteration": dict(n_of=lambda r: 100_000, tags=lambda w: [group_tag(3, r) for r in range(w)]),
    "scale": dict(n_of=lambda r: 100_000, algo=_native.ALGO_ONESHOT, scales=lambda w: [1.0 / (r + 1) for r in range(w)]),
    "cta_cap": dict(n_of=lambda r: 3_000_000, algo=_native.ALGO_TWOSHOT, ctas=lambda w: [8] + [2 * 148 // w] * (w - 1)),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("n_ranks", [2, 4])
def test_disagreement_raises_protocol_error_fast(torch_cuda, group, case, n_ranks):
    torch = torch_cuda
    grp = group(n_ranks)
    c = CASES[case]
    errs, dt = _disagree(torch, grp, c["n_of"], algo=c.get("algo", _native.ALGO_AUTO),
                         tags=c["tags"](n_ranks) if "tags" in c else None,
                         ctas=c["ctas"](n_ranks) if "ctas" in c else None,
                         scales=c["scales"](n_ranks) if "scales" in c else None)
    assert all(isinstance(e, ProtocolError) for e in errs), errs
    assert dt < 1.0, dt
    grp.clear_errors()
    # after the reset the same group reduces correctly
    good, _ = _disagree(torch, grp, lambda r: 100_000)
    assert good == [None] * n_ranks


def test_swapped_group_order_raises(torch_cuda, group):
    """Two equal-size groups issued in different orders on two ranks (the reference's
    frame header group_low check) -> ProtocolError, not silently crossed sums."""
    torch = torch_cuda
    grp = group(2)
    for step in range(2):
        lows = (3, 5) if step == 0 else (5, 3)  # rank 0 sends group 3 then 5, rank 1 the reverse
        errs, _ = _disagree(torch, grp, lambda r: 50_000, tags=[group_tag(lows[0]), group_tag(lows[1])])
        assert all(isinstance(e, ProtocolError) for e in errs), errs
        grp.clear_errors()


def test_matching_tags_pass(torch_cuda, group):
    """Equal (group, iteration) tags on every rank reduce normally."""
    torch = torch_cuda
    grp = group(4)
    errs, _ = _disagree(torch, grp, lambda r: 77_777, tags=[group_tag(11, 5)] * 4)
    assert errs == [None] * 4


def test_absent_peer_times_out(torch_cuda):
    """A rank that never joins: the others raise ProtocolError after the session timeout
    (bounded spins, no hang); the SMs are released."""
    torch = torch_cuda
    grp = LocalGroup(2, device=0, capacity_bytes=1 << 20, timeout=0.5)
    try:
        tensors = [[torch.ones(4096, device="cuda")] for _ in range(2)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        errs = grp.allreduce_fused(tensors, _native.ALGO_ONESHOT, absent=(1,))
        dt = time.perf_counter() - t0
        assert isinstance(errs[0], ProtocolError) and "never reached" in str(errs[0])
        assert 0.4 < dt < 3.0
    finally:
        grp.close()


@pytest.mark.parametrize("n_ranks", [2, 4])
def test_bench_allreduce_local_group(torch_cuda, group, n_ranks):
    """``bench_allreduce`` (allreduce_net.py:414-445 contract) through the real protocol on one
    GPU: one Measurement per size, positive and growing with size, exact sums checked
    inside, and the (a, b) fit of the reference's cost model is positive."""
    from paper_1811_11141_b200 import fit_ab

    grp = group(n_ranks)
    sizes = [4096, 65536, 1 << 20, 4 << 20, 16 << 20]
    ms = grp.bench_allreduce(sizes, repeats=3, warmups=2)
    assert [m.nbytes for m in ms] == sizes and all(m.n_nodes == n_ranks for m in ms)
    assert all(m.seconds > 0 for m in ms)
    assert ms[-1].seconds > ms[0].seconds
    model = fit_ab(ms)
    assert model.a > 0 and model.b > 0
    with pytest.raises(ValueError):
        grp.bench_allreduce([6])
