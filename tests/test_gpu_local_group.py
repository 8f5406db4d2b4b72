"""The real multi-rank protocol on ONE B200: an in-process rank group (``LocalGroup``,
``mgw_comm_create_local``) whose ranks run concurrently on their own streams, so every
barrier, LL header, push store and tag check of the IPC path executes between live
kernels -- the driver's 1-GPU box sees the same device code the NVSwitch ranks run.

Covers: every fused algorithm (fp32 LL / pull one-shot / pull two-shot / push one-shot /
push two-shot; bf16 LL / one-shot / two-shot) through ``mgw_allreduce_fused`` with the
kernels' own pack, bit-exact against the oracle ring (reference fold order,
allreduce_net.py:370-411) for N in {2, 3, 4, 8}; the public ``ring_allreduce`` API with
numpy payloads (reference semantics); the collective tag (allreduce_net.py:340-345):
length, group, iteration, dtype, algorithm-threshold and CTA-cap disagreements raise
ProtocolError on every rank in well under a second; timeouts; error reset; and
``run_emulation`` (Algorithm 2) for fp32 / bf16 / fp64-priced profiles with the gate and
programmatic launch on.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import pytest

from oracle import ring_oracle
from paper_1811_11141_b200 import _native
from paper_1811_11141_b200.allreduce_net import GradientBuffer, LocalGroup, ProtocolError, ring_allreduce

pytestmark = pytest.mark.gpu

ALGOS_F32 = [_native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_PUSH_ONESHOT,
             _native.ALGO_PUSH]
ALGOS_B16 = [_native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT]


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


def fused_exchange(torch, grp, tensors, algo, *, scale=1.0, bf16=False, n_override=None, tags=None):
    """Every rank's fused group exchange on its own thread/stream; returns the per-rank
    exception (None when the rank succeeded)."""
    torch.cuda.synchronize()
    fn_name = "mgw_allreduce_fused_bf16" if bf16 else "mgw_allreduce_fused"

    def body(cfg, sess):
        ts = tensors[cfg.rank]
        rows, off = [], 0
        for t in ts:
            rows.append((t.data_ptr(), t.numel(), off))
            off += t.numel()
        table = _native.DeviceTable(rows)
        try:
            if tags is not None:
                _native.call("mgw_comm_set_group_tag", sess.comm, tags[cfg.rank])
            _native.call(fn_name, sess.comm, table.ptr, table.n, off, ctypes.c_float(scale), algo,
                         sess.stream.cuda_stream)
            sess.stream.synchronize()
            sess.raise_if_failed()
            return None
        except ProtocolError as exc:
            return exc
        finally:
            table.close()
            if tags is not None:
                _native.call("mgw_comm_set_group_tag", sess.comm, 0)

    return grp.run(body)


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
    errs = fused_exchange(torch, group(n_ranks), tensors, algo)
    assert errs == [None] * n_ranks
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
    errs = fused_exchange(torch, group(n_ranks), tensors, algo, scale=scale, bf16=True)
    assert errs == [None] * n_ranks
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
    """AUTO across the LL / one-shot / two-shot / push crossovers, one tensor per rank."""
    torch = torch_cuda
    n = nbytes // 4 + 3
    gen = torch.Generator(device="cuda").manual_seed(n_ranks * 7 + nbytes)
    tensors = [[torch.randn(n, generator=gen, device="cuda")] for _ in range(n_ranks)]
    host = [[t[0].cpu().numpy()] for t in tensors]
    errs = fused_exchange(torch, group(n_ranks), tensors, _native.ALGO_AUTO)
    assert errs == [None] * n_ranks
    _check_f32(tensors, host, [n])


@pytest.mark.parametrize("n_ranks", [2, 3, 4])
def test_ring_allreduce_public_api(torch_cuda, group, n_ranks):
    """The reference call (numpy GradientBuffer in, same object out, in place) on every rank,
    across sizes 0, 1, 17, below N, the LL ceiling and a two-shot bucket; sums exact
    (allreduce_net tests: arange + rank, rank + 1)."""
    grp = group(n_ranks)
    sizes = [0, 1, n_ranks - 1, 17, 1001, 131072, 2_000_003]

    def body(cfg, sess):
        out = []
        for it, n in enumerate(sizes):
            buf = GradientBuffer(3, 5, (np.arange(n, dtype="<f4") % 251) + cfg.rank)
            got = ring_allreduce(buf, cfg, sess, iteration=it)
            assert got is buf
            out.append(buf.values.copy())
        return out

    res = grp.run(body)
    for k, n in enumerate(sizes):
        want = ((np.arange(n, dtype="<f4") % 251) * n_ranks + n_ranks * (n_ranks - 1) / 2).astype("<f4")
        for r in range(n_ranks):
            assert np.array_equal(res[r][k], want), (r, n)


def _mismatch(torch, grp, make, expect_fail=True):
    """Run one exchange per rank whose arguments come from make(rank) -> (n, algo, bf16,
    tag, max_ctas); returns (errors, seconds)."""
    torch.cuda.synchronize()

    def body(cfg, sess):
        n, algo, bf16, tag, ctas = make(cfg.rank)
        x = torch.ones(max(n, 1), dtype=torch.bfloat16 if bf16 else torch.float32, device=sess.device)[:n]
        torch.cuda.synchronize()
        table = _native.DeviceTable([(x.data_ptr(), n, 0)])
        if ctas:
            _native.call("mgw_comm_set_max_ctas", sess.comm, ctas)
        _native.call("mgw_comm_set_group_tag", sess.comm, tag)
        try:
            _native.call("mgw_allreduce_fused_bf16" if bf16 else "mgw_allreduce_fused", sess.comm, table.ptr, 1, n,
                         ctypes.c_float(1.0), algo, sess.stream.cuda_stream)
            sess.stream.synchronize()
            sess.raise_if_failed()
            return None
        except ProtocolError as exc:
            return exc
        finally:
            table.close()
            _native.call("mgw_comm_set_group_tag", sess.comm, 0)
            _native.call("mgw_comm_set_max_ctas", sess.comm, 2 * 148 // cfg.n_workers)

    t0 = time.perf_counter()
    errs = grp.run(body)
    dt = time.perf_counter() - t0
    if expect_fail:
        # every rank saw the disagreement; reset and prove the group still works
        grp.run(lambda cfg, sess: sess.clear_error())
    return errs, dt


CASES = {
    # name: make(rank) -> (n, algo, bf16, group tag, max_ctas)
    "length": lambda r: (100_000 + r, _native.ALGO_AUTO, False, 7, 0),
    "length_ll": lambda r: (1000 + r, _native.ALGO_LL, False, 7, 0),
    "group": lambda r: (100_000, _native.ALGO_AUTO, False, 7 + r, 0),
    "dtype": lambda r: (100_000, _native.ALGO_ONESHOT, r == 1, 7, 0),
    "algorithm": lambda r: (3_000_000, _native.ALGO_ONESHOT if r == 0 else _native.ALGO_TWOSHOT, False, 7, 0),
    "cta_cap": lambda r: (3_000_000, _native.ALGO_TWOSHOT, False, 7, 8 if r == 0 else 0),
    "push_vs_pull": lambda r: (3_000_000, _native.ALGO_PUSH if r == 0 else _native.ALGO_TWOSHOT, False, 7, 0),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("n_ranks", [2, 4])
def test_disagreement_raises_protocol_error_fast(torch_cuda, group, case, n_ranks):
    torch = torch_cuda
    grp = group(n_ranks)
    errs, dt = _mismatch(torch, grp, CASES[case])
    assert all(isinstance(e, ProtocolError) for e in errs), errs
    assert dt < 1.0, dt
    # after the reset the same group reduces correctly
    good, _ = _mismatch(torch, grp, lambda r: (100_000, _native.ALGO_AUTO, False, 9, 0), expect_fail=False)
    assert good == [None] * n_ranks


def test_swapped_group_order_raises(torch_cuda, group):
    """Two equal-size groups issued in different orders on two ranks (reference: frame
    header group_low check) -> ProtocolError, not silently crossed sums."""
    torch = torch_cuda
    grp = group(2)
    torch.cuda.synchronize()

    def body(cfg, sess):
        order = [(3, 12), (5, 12)] if cfg.rank == 0 else [(5, 12), (3, 12)]
        errs = []
        for low, high in order:
            buf = GradientBuffer(low, high, np.ones(50_000, dtype="<f4"))
            try:
                ring_allreduce(buf, cfg, sess)
                errs.append(None)
            except ProtocolError as exc:
                errs.append(exc)
                sess.clear_error()
        return errs

    res = grp.run(body)
    assert all(isinstance(e, ProtocolError) for e in res[0] + res[1]), res


def test_absent_peer_times_out(torch_cuda):
    """A rank that never joins: the others raise ProtocolError after the session timeout
    (bounded spins, no hang)."""
    torch = torch_cuda
    grp = LocalGroup(2, device=0, capacity_bytes=1 << 20, timeout=0.5)
    try:
        for s in grp.sessions:
            _native.call("mgw_comm_set_timeout_ms", s.comm, 500)
        x = torch.ones(4096, device="cuda")
        table = _native.DeviceTable([(x.data_ptr(), 4096, 0)])
        sess = grp.sessions[0]
        t0 = time.perf_counter()
        _native.call("mgw_allreduce_fused", sess.comm, table.ptr, 1, 4096, ctypes.c_float(1.0),
                     _native.ALGO_ONESHOT, sess.stream.cuda_stream)
        sess.stream.synchronize()
        dt = time.perf_counter() - t0
        with pytest.raises(ProtocolError, match="never reached"):
            sess.raise_if_failed()
        assert 0.4 < dt < 3.0
        table.close()
    finally:
        grp.close()


@pytest.mark.parametrize("n_ranks", [2, 4])
@pytest.mark.parametrize("element_bytes", [2, 4, 8])
@pytest.mark.parametrize("gate", [False, True])
def test_run_emulation_local_group(torch_cuda, n_ranks, element_bytes, gate):
    """Algorithm 2 (run_emulation) on every rank with the reference's exact-sum check,
    element_bytes 2 / 4 / 8 (fp32 buffers, as the reference), the fused exchange with
    programmatic launch on, and the peer gate on or off (the gate must wait for the fill)."""
    from paper_1811_11141_b200 import CommModel, find_merge_plan, resnet50_like, run_emulation
    from paper_1811_11141_b200.model_profile import LayerProfile, ModelProfile

    base = resnet50_like(backward_seconds=3e-3, forward_seconds=1e-3)
    profile = ModelProfile(name=base.name, layers=base.layers, forward_time=base.forward_time,
                           element_bytes=element_bytes)
    assert all(isinstance(l, LayerProfile) for l in profile.layers)
    plan = find_merge_plan(profile, CommModel(a=2e-4, b=1e-10))
    grp = LocalGroup(n_ranks, device=0, capacity_bytes=4 * base.total_params, timeout=10.0)
    try:
        if gate:
            for s in grp.sessions:
                _native.call("mgw_comm_set_gate", s.comm, 1)
        reports = grp.run(lambda cfg, sess: run_emulation(profile, plan, cfg, sess, 3, warmup=1, graph=True))
    finally:
        grp.close()
    for r, rep in enumerate(reports):
        assert rep.rank == r and rep.n_workers == n_ranks
        assert rep.verified
        assert rep.allreduce_count == 4 * len([g for g in plan.groups()])
        assert rep.mean_seconds >= 4e-3 * 0.99
