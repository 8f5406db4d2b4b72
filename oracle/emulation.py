"""ORACLE (test infrastructure): CPU restatement of Algorithm 2 for the CPU baseline.

Follows ``run_emulation`` (/root/reference/pkg/src/mgwfbp/allreduce_net.py:463-578):
a compute-agent thread burns ``t_f`` and every ``t_b`` with the reference's
sleep-then-spin ``_delay`` (:448-460) and queues each finished layer; the main
thread pops layers in strictly descending order, packs them (:546) and, when a
group's lowest layer arrives, all-reduces the group with the reference ring
(:370-411) and verifies the exact expected sums (:507, :556).  The N ranks are
simulated in this process (one pthread per rank in the C ring), so the socket
transport is replaced by in-memory segment copies -- strictly cheaper than the
reference's loopback TCP, i.e. a conservative baseline.

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference``.
"""

from __future__ import annotations

import ctypes
import queue
import statistics
import sys
import threading
import time

import numpy as np

from . import ring_oracle


def delay(seconds: float) -> None:
    """allreduce_net.py:448-460: sleep all but ~1.2 ms of long waits, spin the tail."""
    if seconds <= 0.0:
        return
    deadline = time.perf_counter() + seconds
    if seconds >= 0.002:
        slack = seconds - 0.0012
        if slack > 0:
            time.sleep(slack)
    while time.perf_counter() < deadline:
        pass


def _lib():
    lib = ring_oracle._load()
    if lib is None:
        raise RuntimeError("C oracle not built (make -C oracle)")
    if not hasattr(lib, "_fill_bound"):
        lib.oracle_fill_ranks.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_float, ctypes.c_int]
        lib.oracle_fill_ranks.restype = None
        lib._fill_bound = True
    return lib


def ring_seconds(n_ranks: int, nbytes: int, repeats: int = 5, warmups: int = 1) -> float:
    """Median seconds of one oracle ring all-reduce of ``nbytes`` over ``n_ranks``
    simulated ranks (the reference's bench_allreduce protocol, :414-445)."""
    lib = _lib()
    n = nbytes // 4
    bufs = [np.empty(n, dtype="<f4") for _ in range(n_ranks)]
    ptrs = (ctypes.c_void_p * n_ranks)(*[b.ctypes.data for b in bufs])
    times = []
    for r in range(warmups + repeats):
        lib.oracle_fill_ranks(ptrs, n_ranks, 0, n, 1.0, n_ranks)
        t0 = time.perf_counter()
        lib.oracle_ring_allreduce(ptrs, n_ranks, n, n_ranks)
        if r >= warmups:
            times.append(time.perf_counter() - t0)
    return statistics.median(times)


def emulate(profile, plan, n_ranks: int, iterations: int, *, warmup: int = 1, time_budget_s: float | None = None):
    """Run the CPU Algorithm 2; returns (iteration seconds kept, verified)."""
    lib = _lib()
    counts = profile.param_counts()
    t_b = profile.backward_times()
    n_layers = profile.num_layers
    slots, bufs, ptrs = {}, {}, {}
    for low, high in plan.groups():
        rows = ring_oracle.group_rows(counts, low, high)
        total = sum(p for _, p, _ in rows)
        for layer, p, off in rows:
            slots[layer] = (low, off, p)
        bufs[low] = [np.zeros(total, dtype="<f4") for _ in range(n_ranks)]
        ptrs[low] = (ctypes.c_void_p * n_ranks)(*[b.ctypes.data for b in bufs[low]])
    q: "queue.Queue[int]" = queue.Queue()
    done = threading.Event()
    stop = threading.Event()
    walls: list[float] = []

    def agent():
        k = 0
        while not stop.is_set():
            start = time.perf_counter()
            delay(profile.forward_time)
            for layer in range(n_layers, 0, -1):
                if stop.is_set():
                    return
                delay(t_b[layer - 1])
                q.put(layer)
            while not done.wait(0.1):
                if stop.is_set():
                    return
            done.clear()
            walls.append(time.perf_counter() - start)
            k += 1

    verified = True
    old = sys.getswitchinterval()
    sys.setswitchinterval(5e-4)
    th = threading.Thread(target=agent, daemon=True)
    th.start()
    t_begin = time.perf_counter()
    it = 0
    try:
        while it < warmup + iterations:
            for layer in range(n_layers, 0, -1):
                popped = q.get(timeout=120)
                if popped != layer:
                    raise RuntimeError(f"queue discipline broken: expected {layer}, got {popped}")
                low, off, size = slots[layer]
                if size:
                    lib.oracle_fill_ranks(ptrs[low], n_ranks, off, size, float(1 + layer % 5), n_ranks)
                if layer == low:
                    total = len(bufs[low][0])
                    if total and n_ranks > 1:
                        lib.oracle_ring_allreduce(ptrs[low], n_ranks, total, n_ranks)
                    if total:
                        for l2, (lo2, o2, p2) in slots.items():
                            if lo2 == low and p2:
                                want = ring_oracle.emulation_expected(n_ranks, l2) if n_ranks > 1 else float(1 + l2 % 5)
                                seg = bufs[low][0][o2 : o2 + p2]
                                if seg[0] != want or seg[-1] != want:
                                    verified = False
                    if layer == 1:
                        done.set()
            it += 1
            # wait for the agent to log this iteration
            while len(walls) < it and th.is_alive():
                time.sleep(1e-4)
            if time_budget_s is not None and time.perf_counter() - t_begin > time_budget_s and it > warmup:
                break
    finally:
        stop.set()
        done.set()
        sys.setswitchinterval(old)
        th.join(timeout=5.0)
    return walls[warmup:it], verified
