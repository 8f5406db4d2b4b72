"""Host-side multi-process logic on the CPU: the rank-0 rendezvous carrying IPC-handle
payloads (spawned processes, loopback TCP) and the torch.distributed handle exchange used
under torchrun (gloo, world_size 2).  No GPU involved."""

import multiprocessing as mp
import os
import socket

import pytest

from paper_1811_11141_b200 import WorkerConfig, rendezvous
from paper_1811_11141_b200.allreduce_net import _free_port, _segments, exchange_handles_dist


def _rdv_worker(rank, world, port, q):
    payload = bytes([rank]) * 64
    with socket.create_server(("127.0.0.1", 0)) as lst:
        addrs, blobs = rendezvous(rank, world, "127.0.0.1", port, lst.getsockname()[1], timeout=20, payload=payload)
    q.put((rank, addrs, blobs))


def test_rendezvous_distributes_ports_and_handles():
    world = 3
    port = _free_port("127.0.0.1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rdv_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (a, b)) for r, a, b in (q.get(timeout=60) for _ in range(world)))
    for p in procs:
        p.join(timeout=10)
    tables = {tuple(v[0]) for v in got.values()}
    assert len(tables) == 1  # everyone sees the same address table
    (addrs,) = tables
    assert len(set(addrs)) == world
    WorkerConfig(rank=0, n_workers=world, ring_addresses=addrs)  # valid ring view
    for r in range(world):
        assert got[r][1] == [bytes([k]) * 64 for k in range(world)]


def test_rendezvous_without_payload_matches_reference_shape():
    port = _free_port("127.0.0.1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()

    def run(rank):
        return ctx.Process(target=_plain_worker, args=(rank, 2, port, q))

    procs = [run(r) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=60) for _ in range(2)]
    for p in procs:
        p.join(timeout=10)
    assert all(isinstance(t, tuple) and len(t) == 2 for t in res)
    assert res[0] == res[1]


def _plain_worker(rank, world, port, q):
    with socket.create_server(("127.0.0.1", 0)) as lst:
        q.put(rendezvous(rank, world, "127.0.0.1", port, lst.getsockname()[1], timeout=20))


def test_rendezvous_validates_rank():
    with pytest.raises(ValueError):
        rendezvous(2, 2, "127.0.0.1", 1, 1)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        joined = exchange_handles_dist(bytes([0xA0 + rank]) * 64)
        try:
            exchange_handles_dist(b"short")
            bad = None
        except ValueError as exc:
            bad = str(exc)
        q.put((rank, joined, bad))
    finally:
        dist.destroy_process_group()


def test_handle_exchange_over_gloo_world_size_2():
    world = 2
    port = _free_port("127.0.0.1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (j, b)) for r, j, b in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=10)
    want = bytes([0xA0]) * 64 + bytes([0xA1]) * 64
    assert res[0][0] == want and res[1][0] == want
    assert "64 bytes" in res[0][1]


def test_segments_match_reference_split():
    assert _segments(10, 4) == ([3, 3, 2, 2], [0, 3, 6, 8])
    assert _segments(1, 8)[0] == [1, 0, 0, 0, 0, 0, 0, 0]
    assert _segments(0, 3) == ([0, 0, 0], [0, 0, 0])


def test_auto_algorithm_rule_mirrors_the_native_choice():
    """allreduce_net._algo_for (transport accounting) follows pick_fused_algo's rule."""
    from types import SimpleNamespace

    from paper_1811_11141_b200 import _native
    from paper_1811_11141_b200.allreduce_net import _algo_for

    def algo(world, nbytes):
        return _algo_for(SimpleNamespace(config=SimpleNamespace(n_workers=world)), nbytes // 4, fused=True)

    assert algo(2, 4096) == algo(2, 256 << 10) == _native.ALGO_LL
    assert algo(2, 512 << 10) == algo(2, 16 << 20) == _native.ALGO_LL128_ONESHOT
    assert algo(2, 32 << 20) == algo(2, 128 << 20) == _native.ALGO_LL128
    assert algo(2, 256 << 20) == _native.ALGO_PUSH and algo(2, 2 << 30) == _native.ALGO_TWOSHOT
    assert algo(4, 128 << 10) == _native.ALGO_LL and algo(4, 256 << 10) == algo(4, 1 << 20) == _native.ALGO_LL128_ONESHOT
    assert algo(4, 2 << 20) == algo(4, 64 << 20) == _native.ALGO_LL128
    assert algo(4, 128 << 20) == _native.ALGO_PUSH
    assert algo(8, 256 << 10) == _native.ALGO_LL and algo(8, 512 << 10) == _native.ALGO_PUSH_ONESHOT
    assert algo(8, 1 << 20) == _native.ALGO_LL128 and algo(8, 2 << 30) == _native.ALGO_TWOSHOT
    assert algo(8, 20 << 20) == _native.ALGO_PUSH
