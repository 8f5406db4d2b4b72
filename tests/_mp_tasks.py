"""Picklable per-rank tasks for run_workers (spawned processes import this module)."""

import numpy as np

from paper_1811_11141_b200 import GradientBuffer, ring_allreduce


def sum_task(config, session):
    vals = np.arange(23, dtype="<f4") + config.rank
    buf = GradientBuffer(1, 1, vals)
    assert ring_allreduce(buf, config, session) is buf
    n = config.n_workers
    assert np.array_equal(buf.values, np.arange(23, dtype="<f4") * n + n * (n - 1) / 2)
    buf2 = GradientBuffer(1, 1, np.ones(5, dtype="<f4"))
    ring_allreduce(buf2, config, session)
    assert np.array_equal(buf2.values, np.full(5, n, dtype="<f4"))
    return session.counters.frames_sent


def single_element_task(config, session):
    buf = GradientBuffer(1, 1, np.array([float(config.rank + 1)], dtype="<f4"))
    ring_allreduce(buf, config, session)
    n = config.n_workers
    return bool(buf.values[0] == n * (n + 1) / 2)


def mismatched_task(config, session):
    size = 8 if config.rank == 0 else 12
    ring_allreduce(GradientBuffer(1, 1, np.zeros(size, dtype="<f4")), config, session)
    return True


def collective_task(config, session):
    verdicts = []
    for elements in (1, 17, 1_000_000, 5_000_003):
        buf = GradientBuffer(1, 1, np.full(elements, float(config.rank + 1), dtype="<f4"))
        ring_allreduce(buf, config, session)
        n = config.n_workers
        verdicts.append(bool((buf.values == n * (n + 1) / 2).all()))
    return verdicts


def random_task(config, session, *, arrays):
    """Reduce the golden per-rank inputs through the real IPC path."""
    import torch

    out = {}
    for key, vals in arrays[config.rank].items():
        buf = GradientBuffer(1, 1, vals.copy())
        ring_allreduce(buf, config, session)
        out[key] = buf.values.copy()
        t = torch.from_numpy(vals.copy()).to(session.device)
        ring_allreduce(GradientBuffer(1, 1, t), config, session)
        out[key + "_tensor"] = t.cpu().numpy()
    return out


def emulate_task(config, session, *, profile, plan, fused, graph):
    from paper_1811_11141_b200 import run_emulation

    return run_emulation(profile, plan, config, session, 3, warmup=1, fused=fused, graph=graph)


def every_algorithm_task(config, session, *, arrays):
    """Each algorithm (fused LL / one-shot / two-shot, unfused one-shot / two-shot) on the
    golden inputs through the real IPC path; returns the reduced bits per (size, algo)."""
    import ctypes

    import torch

    from paper_1811_11141_b200 import _native

    out = {}
    h = session.stream.cuda_stream
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        for key, vals in arrays[config.rank].items():
            n = vals.size
            for name, algo in (("ll", _native.ALGO_LL), ("one", _native.ALGO_ONESHOT), ("two", _native.ALGO_TWOSHOT),
                               ("push", _native.ALGO_PUSH), ("push1", _native.ALGO_PUSH_ONESHOT),
                               ("ll128", _native.ALGO_LL128), ("ll128_1", _native.ALGO_LL128_ONESHOT)):
                t = torch.from_numpy(vals.copy()).to(session.device)
                table = _native.DeviceTable([(t.data_ptr(), n, 0)])
                _native.call("mgw_allreduce_fused", session.comm, table.ptr, 1, n, ctypes.c_float(1.0), algo, h)
                session.stream.synchronize()
                session.raise_if_failed()
                out[f"{key}_fused_{name}"] = t.cpu().numpy()
                table.close()
            for name, algo in (("one", _native.ALGO_ONESHOT), ("two", _native.ALGO_TWOSHOT)):
                t = torch.from_numpy(vals.copy()).to(session.device)
                table = _native.DeviceTable([(t.data_ptr(), n, 0)])
                _native.call("mgw_comm_pack", session.comm, table.ptr, 1, n, ctypes.c_float(1.0), h)
                _native.call("mgw_allreduce", session.comm, n, algo, h)
                _native.call("mgw_unpack", table.ptr, 1, session.result_ptr(), n, h)
                session.stream.synchronize()
                session.raise_if_failed()
                out[f"{key}_plain_{name}"] = t.cpu().numpy()
                table.close()
            # peer gate on: the same bits, one extra one-warp kernel per collective
            _native.call("mgw_comm_set_gate", session.comm, 1)
            for name, algo in (("ll", _native.ALGO_LL), ("two", _native.ALGO_TWOSHOT)):
                t = torch.from_numpy(vals.copy()).to(session.device)
                table = _native.DeviceTable([(t.data_ptr(), n, 0)])
                _native.call("mgw_allreduce_fused", session.comm, table.ptr, 1, n, ctypes.c_float(1.0), algo, h)
                session.stream.synchronize()
                session.raise_if_failed()
                out[f"{key}_gate_{name}"] = t.cpu().numpy()
                table.close()
            _native.call("mgw_comm_set_gate", session.comm, 0)
    return out


def autograd_task(config, session, *, algo=0, deferred=False, gate=False):
    """Two+ ranks with different data: merged-gradient sync leaves averaged gradients equal,
    bit for bit, to the oracle ring over the per-rank gradients.  The model is elementwise so
    its backward is deterministic (cuBLAS split-K GEMMs are not, run to run)."""
    import torch

    from paper_1811_11141_b200 import MergePlan
    from paper_1811_11141_b200.autograd import MergedGradientSync, trainable_parameters

    class Elementwise(torch.nn.Module):
        def __init__(self):
            super().__init__()
            g = torch.Generator().manual_seed(0)
            self.w = torch.nn.ParameterList(
                [torch.nn.Parameter(torch.randn(n, generator=g)) for n in (16448, 257, 2570, 10)])

        def forward(self, xs):
            return sum((w * x).sin().square().sum() for w, x in zip(self.w, xs))

    net = Elementwise().to(session.device)
    g = torch.Generator(device=session.device).manual_seed(1000 + config.rank)
    xs = [torch.randn(w.numel(), device=session.device, generator=g) for w in net.w]
    params = trainable_parameters(net)
    net.zero_grad(set_to_none=False)
    net(xs).backward()
    local = [p.grad.detach().cpu().numpy().copy() for p in params]
    net.zero_grad(set_to_none=False)
    net(xs).backward()
    again = [p.grad.detach().cpu().numpy().copy() for p in params]
    sync = MergedGradientSync(params, MergePlan(frozenset({2, 4}), 4), comm=session.comm, world=config.n_workers,
                              algo=algo, sync_after_backward=deferred, gate=gate, priority=-1 if gate else 0)
    net.zero_grad(set_to_none=False)
    net(xs).backward()
    if deferred:  # groups not launched yet: the synced backward's own gradients
        torch.cuda.synchronize()
        third = [p.grad.detach().cpu().numpy().copy() for p in params]
        local = third
    sync.finish()
    torch.cuda.synchronize()
    session.raise_if_failed()
    sync.close()
    deterministic = all((a.view("<u4") == b.view("<u4")).all() for a, b in zip(local, again))
    return local, [p.grad.detach().cpu().numpy() for p in params], deterministic


def sizes_task(config, session, *, sizes, algos):
    """Seeded random payloads of several sizes split into two rows, through each fused
    algorithm; returns inputs and outputs for a host-side oracle comparison."""
    import ctypes

    import numpy as np
    import torch

    from paper_1811_11141_b200 import _native

    out = {}
    h = session.stream.cuda_stream
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        for n in sizes:
            vals = np.random.default_rng(7 * n + config.rank).standard_normal(n).astype("<f4")
            out[("in", n)] = vals
            for algo in algos:
                a = torch.from_numpy(vals[:257].copy()).to(session.device)
                b = torch.from_numpy(vals[257:].copy()).to(session.device)
                table = _native.DeviceTable([(a.data_ptr(), 257, 0), (b.data_ptr(), n - 257, 257)])
                _native.call("mgw_allreduce_fused", session.comm, table.ptr, 2, n, ctypes.c_float(1.0), algo, h)
                session.stream.synchronize()
                session.raise_if_failed()
                out[(algo, n)] = np.concatenate([a.cpu().numpy(), b.cpu().numpy()])
                table.close()
    return out


def replan_task(config, session, *, iterations=4):
    """Live group-exchange spans of real overlapped iterations feed the online planner."""
    import torch

    from paper_1811_11141_b200 import MergePlan, find_merge_plan, resnet50_like
    from paper_1811_11141_b200.overlap import OverlappedIteration
    from paper_1811_11141_b200.replan import OnlinePlanner, observe_iteration

    profile = resnet50_like(backward_seconds=0.00972, forward_seconds=0.00464)
    plan = MergePlan(frozenset(), profile.num_layers)
    planner = OnlinePlanner(profile, config.n_workers, plan=plan, min_samples=16)
    with torch.cuda.device(session.device):
        it = OverlappedIteration(profile, plan, comm=session.comm, rank=config.rank, world=config.n_workers,
                                 device=session.device, fused=True)
        try:
            for _ in range(iterations):
                it.run()
                observe_iteration(planner, it)
            ok = it.verify()
        finally:
            it.close()
    session.raise_if_failed()
    new = planner.update()
    m = planner.model
    return {"verified": ok, "samples": len(planner.samples), "a": m.a, "b": m.b,
            "consistent": (new or planner.plan) == find_merge_plan(profile, m)}


def bf16_task(config, session, *, sizes):
    """bf16 payloads (seeded per rank) through ring_allreduce (AUTO) and each explicit
    algorithm of mgw_allreduce_fused_bf16; inputs and outputs as uint16 bit patterns."""
    import ctypes

    import numpy as np
    import torch

    from paper_1811_11141_b200 import GradientBuffer, _native

    out = {}
    h = session.stream.cuda_stream
    for n in sizes:
        g = torch.Generator().manual_seed(11 * n + config.rank)
        vals = (torch.randn(n, generator=g) * 4).to(torch.bfloat16)
        out[("in", n)] = vals.view(torch.int16).numpy().view(np.uint16).copy()
        t = vals.to(session.device)
        ring_allreduce(GradientBuffer(1, 1, t), config, session)
        out[("auto", n)] = t.view(torch.int16).cpu().numpy().view(np.uint16)
        algos = [("one", _native.ALGO_ONESHOT), ("two", _native.ALGO_TWOSHOT), ("ll128", _native.ALGO_LL128)]
        if n <= 131072:
            algos.append(("ll", _native.ALGO_LL))
        for name, algo in algos:
            t = vals.to(session.device)
            table = _native.DeviceTable([(t.data_ptr(), n, 0)])
            with torch.cuda.device(session.device):
                session.stream.wait_stream(torch.cuda.current_stream(session.device))
                _native.call("mgw_allreduce_fused_bf16", session.comm, table.ptr, 1, n, ctypes.c_float(0.5), algo, h)
                session.stream.synchronize()
            session.raise_if_failed()
            out[(name, n)] = t.view(torch.int16).cpu().numpy().view(np.uint16)
            table.close()
    out["bytes_received"] = session.counters.payload_bytes_received
    return out


def autograd_bf16_task(config, session):
    """bf16 parameters: merged-gradient sync moves bf16, folds in fp32, averages."""
    import numpy as np
    import torch

    from paper_1811_11141_b200 import MergePlan
    from paper_1811_11141_b200.autograd import MergedGradientSync, trainable_parameters

    g = torch.Generator().manual_seed(0)
    ws = [torch.nn.Parameter(torch.randn(n, generator=g).to(torch.bfloat16).to(session.device))
          for n in (16448, 257, 2570, 10)]
    g2 = torch.Generator(device=session.device).manual_seed(1000 + config.rank)
    xs = [torch.randn(w.numel(), device=session.device, generator=g2).to(torch.bfloat16) for w in ws]

    def loss():
        return sum((w * x).float().sin().square().sum() for w, x in zip(ws, xs))

    for w in ws:
        w.grad = None
    loss().backward()
    local = [w.grad.view(torch.int16).cpu().numpy().view(np.uint16).copy() for w in ws]
    for w in ws:
        w.grad = None
    sync = MergedGradientSync(ws, MergePlan(frozenset({2, 4}), 4), comm=session.comm, world=config.n_workers,
                              scale=1.0 / config.n_workers)
    loss().backward()
    sync.finish()
    torch.cuda.synchronize()
    session.raise_if_failed()
    sync.close()
    return local, [w.grad.view(torch.int16).cpu().numpy().view(np.uint16).copy() for w in ws]


def dtype_mismatch_task(config, session):
    """Rank 0 reduces bf16, the others fp32, same element count: a protocol error."""
    import torch

    from paper_1811_11141_b200 import GradientBuffer

    dtype = torch.bfloat16 if config.rank == 0 else torch.float32
    t = torch.ones(1000, dtype=dtype, device=session.device)
    ring_allreduce(GradientBuffer(1, 1, t), config, session)
    return True


def absent_peer_task(config, session):
    """Rank 0 enters a collective that rank 1 never joins: a bounded device wait ends in a
    ProtocolError (no hang); rank 1 outlives the 2 s device timeout, then leaves."""
    import time

    from paper_1811_11141_b200 import _native

    _native.call("mgw_comm_set_timeout_ms", session.comm, 2000)
    if config.rank != 0:
        time.sleep(5.0)
        return "absent"
    ring_allreduce(GradientBuffer(1, 1, np.ones(4096, dtype="<f4")), config, session)
    return "completed"


def stress_task(config, session, *, iterations=300, seed=2024, only=None, max_n=1 << 21):
    """A seeded stream of collectives with random sizes, row splits, dtypes and algorithms
    (the same on every rank), back to back on one communicator: integer-valued payloads
    must come back exactly.  Exercises slot-parity / LL-area / gather-area reuse across
    algorithm switches.  Returns the number of failures and the first few."""
    import ctypes

    import numpy as np
    import torch

    from paper_1811_11141_b200 import _native

    rng = np.random.default_rng(seed)
    n_ranks = config.n_workers
    algos_f32 = [_native.ALGO_AUTO, _native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_PUSH,
                 _native.ALGO_PUSH_ONESHOT, _native.ALGO_LL128, _native.ALGO_LL128_ONESHOT]
    algos_b16 = [_native.ALGO_AUTO, _native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_LL128,
                 _native.ALGO_LL128_ONESHOT]
    if only is not None:  # a restricted algorithm set (e.g. the LL128 kernels only)
        algos_f32 = [a for a in algos_f32 if a in only]
        algos_b16 = [a for a in algos_b16 if a in only]
    h = session.stream.cuda_stream
    failures = []
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        for it in range(iterations):
            bf16 = bool(rng.random() < 0.25)
            n = int(rng.choice([1, 7, 63, 1000, 4097]) if rng.random() < 0.3 else rng.integers(1, max_n))
            if bf16:
                algo = int(rng.choice(algos_b16))
            else:
                algo = int(rng.choice(algos_f32))
            if algo == _native.ALGO_LL:
                n = min(n, 262144 * (2 if bf16 else 1))
            cuts = sorted(set(int(c) for c in rng.integers(0, n + 1, size=2)))
            bounds = [0] + [c for c in cuts if 0 < c < n] + [n]
            dtype = torch.bfloat16 if bf16 else torch.float32
            idx = torch.arange(n, device=session.device)
            pattern = (idx % 5).to(torch.float32)
            # fp32: an iteration-dependent offset, so a stale line of an earlier call in the
            # same area can never pass for this call's data
            it_off = 0.0 if bf16 else 16.0 * (it % 11)
            x = (pattern + float(config.rank + 1) + it_off).to(dtype)
            rows = []
            views = []
            for lo, hi in zip(bounds[:-1], bounds[1:]):
                v = x[lo:hi].clone()  # separate allocations: the rows live in different tensors
                views.append(v)
                rows.append((v.data_ptr(), hi - lo, lo))
            table = _native.DeviceTable(rows)
            fn = "mgw_allreduce_fused_bf16" if bf16 else "mgw_allreduce_fused"
            _native.call(fn, session.comm, table.ptr, len(rows), n, ctypes.c_float(1.0), algo, h)
            got = torch.cat(views).float()
            want = pattern * n_ranks + n_ranks * (n_ranks + 1) / 2 + n_ranks * it_off
            session.stream.synchronize()
            table.close()
            if not torch.equal(got, want):
                bad = int((got != want).sum())
                failures.append((it, n, algo, bf16, bad))
    session.raise_if_failed()
    return len(failures), failures[:5]


def empty_and_tiny_task(config, session):
    """Zero-length buffers are still collective (the reference's ring runs its rounds on
    empty segments); 1..N-1 elements leave some reference segments empty."""
    import torch

    out = []
    empty = GradientBuffer(1, 1, np.zeros(0, dtype="<f4"))
    assert ring_allreduce(empty, config, session) is empty and len(empty) == 0
    n = config.n_workers
    for size in range(1, n + 2):
        buf = GradientBuffer(1, 1, np.full(size, float(config.rank + 1), dtype="<f4"))
        ring_allreduce(buf, config, session)
        out.append(bool((buf.values == n * (n + 1) / 2).all()))
        t = torch.full((size,), float(config.rank + 1), dtype=torch.bfloat16, device=session.device)
        ring_allreduce(GradientBuffer(1, 1, t), config, session)
        out.append(bool((t.float() == n * (n + 1) / 2).all()))
    # and the next collective after them is still in step
    buf = GradientBuffer(1, 1, np.arange(23, dtype="<f4") + config.rank)
    ring_allreduce(buf, config, session)
    out.append(bool(np.array_equal(buf.values, np.arange(23, dtype="<f4") * n + n * (n - 1) / 2)))
    return out


def _timed_collective(config, session, buf_values, layer_low=1, iteration=0):
    """One ring_allreduce; returns (seconds, error text or None)."""
    import time

    from paper_1811_11141_b200 import ProtocolError

    t0 = time.perf_counter()
    try:
        ring_allreduce(GradientBuffer(layer_low, layer_low, buf_values), config, session, iteration=iteration)
        return time.perf_counter() - t0, None
    except ProtocolError as exc:
        return time.perf_counter() - t0, str(exc)


def cta_cap_mismatch_task(config, session):
    """Rank 0 caps its collectives at 8 CTAs, the others keep the default: the grids differ,
    so the collective tags differ at the first barrier (allreduce_net.py:340-345)."""
    from paper_1811_11141_b200 import _native

    _native.call("mgw_comm_set_timeout_ms", session.comm, 20000)
    if config.rank == 0:
        _native.call("mgw_comm_set_max_ctas", session.comm, 8)
    return _timed_collective(config, session, np.ones(3_000_000, dtype="<f4"))


def threshold_mismatch_task(config, session):
    """Rank 0 disables LL (ll_max 0) and the one-shot (oneshot_max 0): its AUTO choice for a
    64 KiB and a 2 MiB bucket differs from its peers' -> ProtocolError, not crossed data."""
    from paper_1811_11141_b200 import _native

    _native.call("mgw_comm_set_timeout_ms", session.comm, 20000)
    if config.rank == 0:
        _native.call("mgw_comm_set_ll_max", session.comm, 0)
        _native.call("mgw_comm_set_oneshot_max", session.comm, 0)
    return [_timed_collective(config, session, np.ones(16384, dtype="<f4"))]


def swapped_groups_task(config, session):
    """Two equal-size merge groups issued in opposite orders on rank 0 and the others: the
    group tag (head layer) differs at the barrier -> ProtocolError on every rank."""
    from paper_1811_11141_b200 import _native

    _native.call("mgw_comm_set_timeout_ms", session.comm, 20000)
    order = (3, 5) if config.rank == 0 else (5, 3)
    return _timed_collective(config, session, np.ones(100_000, dtype="<f4"), layer_low=order[0])


def iteration_mismatch_task(config, session):
    """Same group, different iteration numbers (the reference header's iteration field)."""
    from paper_1811_11141_b200 import _native

    _native.call("mgw_comm_set_timeout_ms", session.comm, 20000)
    return _timed_collective(config, session, np.ones(5000, dtype="<f4"), layer_low=2, iteration=config.rank)


def emulate_bf16_task(config, session, *, profile, plan):
    """run_emulation on bf16 gradients (bf16 wire, fp32 accumulation) with the reference's
    exact-sum verification."""
    import torch

    from paper_1811_11141_b200 import run_emulation

    rep = run_emulation(profile, plan, config, session, 3, warmup=1, graph=True, dtype=torch.bfloat16)
    return rep.verified, rep.allreduce_count


def wide_push_task(config, session, *, n32, n16):
    """Buckets above the wide-grid threshold (push two-shot at 512 CTAs, a second partial
    wave): fp32 in three ragged rows and bf16, both on the push two-shot, each rank
    regenerating every rank's seeded input to check its result against the oracle in place
    (the arrays are too large to ship back).  Returns mismatch counts."""
    import ctypes

    import numpy as np
    import torch

    from oracle import ring_oracle
    from paper_1811_11141_b200 import _native

    h = session.stream.cuda_stream
    n = config.n_workers
    out = {}
    ins = [np.random.default_rng(1000 + r).standard_normal(n32).astype("<f4") for r in range(n)]
    want = ring_oracle.ring_allreduce(ins)[0]
    cuts = [0, 257, 257 + n32 // 3 + 1, n32]
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        t = torch.from_numpy(ins[config.rank]).to(session.device)
        parts = [t[cuts[i]:cuts[i + 1]] for i in range(3)]
        table = _native.DeviceTable([(p.data_ptr(), p.numel(), cuts[i]) for i, p in enumerate(parts)])
        _native.call("mgw_allreduce_fused", session.comm, table.ptr, 3, n32, ctypes.c_float(1.0), _native.ALGO_PUSH, h)
        session.stream.synchronize()
        session.raise_if_failed()
        out["f32_bad"] = int(np.count_nonzero(t.cpu().numpy().view("<u4") != want.view("<u4")))
        table.close()
    del ins, want
    ins16 = []
    for r in range(n):
        g = torch.Generator().manual_seed(77 + r)
        ins16.append((torch.randn(n16, generator=g) * 4).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16))
    want16 = ring_oracle.ring_allreduce_bf16(ins16, scale=0.5)
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        t = torch.from_numpy(ins16[config.rank].view(np.int16).copy()).view(torch.bfloat16).to(session.device)
        table = _native.DeviceTable([(t.data_ptr(), n16, 0)])
        _native.call("mgw_allreduce_fused_bf16", session.comm, table.ptr, 1, n16, ctypes.c_float(0.5),
                     _native.ALGO_PUSH, h)
        session.stream.synchronize()
        session.raise_if_failed()
        got = t.view(torch.int16).cpu().numpy().view(np.uint16)
        out["b16_bad"] = int(np.count_nonzero(got != want16))
        table.close()
    return out


def algo_mismatch_task(config, session):
    """Rank 0 runs the LL128 two-shot, the others the push two-shot, on the same 8 MB
    bucket: LL128's line polls meet the push barrier words (and the LL header the push
    barrier polls for) -> ProtocolError on every rank, no timeout."""
    import ctypes
    import time

    import torch

    from paper_1811_11141_b200 import ProtocolError, _native

    _native.call("mgw_comm_set_timeout_ms", session.comm, 20000)
    n = 2_000_000
    algo = _native.ALGO_LL128 if config.rank == 0 else _native.ALGO_PUSH
    h = session.stream.cuda_stream
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        t = torch.ones(n, device=session.device)
        table = _native.DeviceTable([(t.data_ptr(), n, 0)])
        t0 = time.perf_counter()
        try:
            _native.call("mgw_allreduce_fused", session.comm, table.ptr, 1, n, ctypes.c_float(1.0), algo, h)
            session.stream.synchronize()
            session.raise_if_failed()
            return time.perf_counter() - t0, None
        except ProtocolError as exc:
            return time.perf_counter() - t0, str(exc)
        finally:
            table.close()
