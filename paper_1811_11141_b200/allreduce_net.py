"""The reference's data-path API, served by the B200 NVLink path.

Drop-in for ``/root/reference/pkg/src/mgwfbp/allreduce_net.py``: the same
names, signatures, argument meanings and error behaviour, with the loopback
TCP ring replaced by sm_100a kernels over CUDA-IPC peer memory.

=====================  ============================================  =========================
name                   B200 implementation                            reference
=====================  ============================================  =========================
``ProtocolError``      device error word -> exception                 :57-58
``WorkerConfig``       + optional ``device`` (default: rank)           :61-95
``GradientBuffer``     numpy ``<f4`` (H2D/D2H per call) or a CUDA      :98-120
                       float32 tensor (zero copy)
``TransportCounters``  NVLink payload bytes pulled / served            :123-131
``EmulationReport``    + measured ``compute_seconds``/``t_c_no``       :134-150
``rendezvous``         rank-0 TCP meeting point, now also carrying     :180-225
                       each rank's 64-byte CUDA-IPC handle
``RingSession``        owns the native communicator (IPC buckets,      :228-275
                       flags, peer mappings) and the comm stream
``_segments``          identical split (fixes the fold order)          :360-367
``ring_allreduce``     K1 pack -> K2/K3 -> K4 unpack, in place         :370-411
``bench_allreduce``    CUDA-event median per size (+ bus GB/s)         :414-445
``run_emulation``      Algorithm 2 as a native stream schedule         :463-578
``open_ring``          IPC rendezvous + peer mapping                   :581-605
``run_workers``        spawn one process per GPU                       :622-683
``bench_local``        ``run_workers`` + ``bench_allreduce``           :694-712
``emulate_local``      ``run_workers`` + ``run_emulation``             :715-734
=====================  ============================================  =========================

Transport-specific semantics that necessarily change: ``chunk_elements`` no
longer frames anything (kept for signature compatibility), and the counters
report NVLink bytes instead of TCP frames; see DESIGN.md.  There is no CPU
fallback: without the native library or a CUDA device every data-path call
raises.
"""

from __future__ import annotations

import ctypes
import queue
import socket
import statistics
import struct
import time
import traceback
from dataclasses import dataclass, field
from functools import partial
from multiprocessing import get_context

import numpy as np

from . import _native
from ._native import ProtocolError
from .comm_model import Measurement
from .merge_planner import MergePlan
from .model_profile import ModelProfile

__all__ = [
    "DEFAULT_CAPACITY_BYTES",
    "EmulationReport",
    "GradientBuffer",
    "LocalGroup",
    "ProtocolError",
    "RingSession",
    "TransportCounters",
    "WorkerConfig",
    "bench_allreduce",
    "bench_local",
    "emulate_local",
    "open_ring",
    "open_session_dist",
    "enable_nvls",
    "rendezvous",
    "ring_allreduce",
    "run_emulation",
    "run_workers",
]

_F32 = np.dtype("<f4")
_DEFAULT_TIMEOUT = 60.0
DEFAULT_CAPACITY_BYTES = 256 << 20  # per slot; 2 slots + result per rank


@dataclass(frozen=True)
class WorkerConfig:
    """One rank's view of the group.

    ``ring_addresses`` are the ranks' rendezvous endpoints in rank order (kept
    unique as in the reference); ``device`` is the CUDA device of this rank.
    """

    rank: int
    n_workers: int
    ring_addresses: tuple[tuple[str, int], ...]
    chunk_elements: int = 1 << 22
    device: int | None = None

    def __post_init__(self) -> None:
        if not isinstance(self.n_workers, int) or self.n_workers < 2:
            raise ValueError(f"n_workers must be an int >= 2, got {self.n_workers!r}")
        if not isinstance(self.rank, int) or not 0 <= self.rank < self.n_workers:
            raise ValueError(f"rank must lie in [0, {self.n_workers}), got {self.rank!r}")
        addrs = tuple((h, int(p)) for h, p in self.ring_addresses)
        object.__setattr__(self, "ring_addresses", addrs)
        if len(addrs) != self.n_workers:
            raise ValueError("need exactly one address per rank")
        if len(set(addrs)) != self.n_workers:
            raise ValueError("ring addresses must be unique")
        if not isinstance(self.chunk_elements, int) or self.chunk_elements < 1:
            raise ValueError(f"chunk_elements must be an int >= 1, got {self.chunk_elements!r}")
        if self.n_workers > _native.MAX_RANKS:
            raise ValueError(f"at most {_native.MAX_RANKS} ranks share one NVSwitch domain here")

    @property
    def right_rank(self) -> int:
        return (self.rank + 1) % self.n_workers

    @property
    def left_rank(self) -> int:
        return (self.rank - 1) % self.n_workers

    @property
    def device_index(self) -> int:
        return self.rank if self.device is None else self.device


def _is_torch_tensor(x) -> bool:
    return type(x).__module__.split(".")[0] == "torch"


class GradientBuffer:
    """Flat fp32 payload of the layer span ``[layer_low, layer_high]``.

    ``values`` is a contiguous little-endian float32 numpy copy (reference
    semantics) or, zero-copy, a contiguous CUDA float32 torch tensor -- or a bf16 one
    (bf16 on the wire, fp32 accumulation, ``mgw_allreduce_fused_bf16``).
    """

    __slots__ = ("layer_low", "layer_high", "values")

    def __init__(self, layer_low: int, layer_high: int, values) -> None:
        if not 1 <= layer_low <= layer_high:
            raise ValueError(f"bad layer range [{layer_low}, {layer_high}]")
        self.layer_low = layer_low
        self.layer_high = layer_high
        if _is_torch_tensor(values):
            import torch

            if values.dtype not in (torch.float32, torch.bfloat16) or values.dim() != 1 or not values.is_contiguous():
                raise ValueError("tensor payloads must be contiguous 1-D float32 or bfloat16")
            self.values = values
        else:
            self.values = np.ascontiguousarray(values, dtype=_F32)

    def __len__(self) -> int:
        return int(self.values.shape[0])

    @classmethod
    def for_group(cls, profile: ModelProfile, layer_low: int, layer_high: int) -> "GradientBuffer":
        """Zero-filled buffer holding exactly the group's parameters."""
        if layer_high > profile.num_layers:
            raise ValueError(f"layer {layer_high} outside profile of {profile.num_layers}")
        total = sum(profile.param_counts()[layer_low - 1 : layer_high])
        return cls(layer_low, layer_high, np.zeros(total, dtype=_F32))


@dataclass
class TransportCounters:
    """NVLink traffic of this rank.  ``rounds`` = barrier phases (1 one-shot,
    2 two-shot); ``frames_*`` = collectives; ``payload_bytes_received`` = bytes
    this rank pulled from peers, ``payload_bytes_sent`` = bytes peers pulled
    from this rank."""

    rounds: int = 0
    frames_sent: int = 0
    frames_received: int = 0
    payload_bytes_sent: int = 0
    payload_bytes_received: int = 0


@dataclass(frozen=True)
class EmulationReport:
    """One rank's measured Algorithm-2 run (reference fields first).

    ``iteration_seconds``/``compute_seconds``/``t_c_no_seconds`` are CUDA-event
    spans per kept iteration; ``group_comm_seconds`` maps each sending group's
    head layer to its mean pack+all-reduce+unpack span.
    """

    rank: int
    n_workers: int
    iteration_seconds: tuple[float, ...]
    mean_seconds: float
    stddev_seconds: float
    group_comm_seconds: dict[int, float]
    verified: bool
    allreduce_count: int
    compute_seconds: tuple[float, ...] = ()
    t_c_no_seconds: tuple[float, ...] = ()
    # Gantt rows (layer, kind, start_s, end_s) of the last iteration, measured by the
    # kernels' own stamps (Timeline.events, schedule_sim.py:88-100)
    events: tuple[tuple[int, str, float, float], ...] = ()


# ----------------------------------------------------------------- bootstrap


def _free_port(host: str) -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind((host, 0))
        return s.getsockname()[1]


def _recv_exact(sock: socket.socket, n: int, who: str) -> bytes:
    chunks, got = [], 0
    while got < n:
        piece = sock.recv(n - got)
        if not piece:
            raise ProtocolError(f"{who}: peer closed the connection")
        chunks.append(piece)
        got += len(piece)
    return b"".join(chunks)


def _connect_retry(address: tuple[str, int], timeout: float, who: str) -> socket.socket:
    deadline = time.monotonic() + timeout
    while True:
        try:
            return socket.create_connection(address, timeout=2.0)
        except OSError:
            if time.monotonic() > deadline:
                raise ProtocolError(f"{who}: cannot reach {address[0]}:{address[1]}")
            time.sleep(0.02)


_HELLO = struct.Struct("<II")


def rendezvous(
    rank: int,
    n_workers: int,
    host: str,
    base_port: int,
    data_port: int,
    *,
    timeout: float = 30.0,
    payload: bytes | None = None,
):
    """Rank-0 meeting point (allreduce_net.py:180-225).

    Every rank reports ``(rank, data_port[, payload])``; rank 0 answers with the
    full table.  Returns the address table, or ``(addresses, payloads)`` when a
    fixed-size ``payload`` (the 64-byte CUDA-IPC handle) rides along.
    """
    if not 0 <= rank < n_workers:
        raise ValueError(f"rank {rank} outside [0, {n_workers})")
    who = f"rank {rank}"
    extra = b"" if payload is None else bytes(payload)
    width = len(extra)
    if rank == 0:
        ports = [0] * n_workers
        blobs = [b""] * n_workers
        ports[0], blobs[0] = data_port, extra
        seen = {0}
        conns: list[socket.socket] = []
        with socket.create_server((host, base_port), backlog=n_workers) as srv:
            srv.settimeout(timeout)
            try:
                for _ in range(n_workers - 1):
                    try:
                        conn, _ = srv.accept()
                    except socket.timeout:
                        raise ProtocolError(f"{who}: only {len(seen)} of {n_workers} ranks joined the rendezvous")
                    conns.append(conn)
                    conn.settimeout(timeout)
                    peer, port = _HELLO.unpack(_recv_exact(conn, _HELLO.size, who))
                    blob = _recv_exact(conn, width, who) if width else b""
                    if not 1 <= peer < n_workers or peer in seen:
                        raise ProtocolError(f"{who}: bad or duplicate rendezvous rank {peer}")
                    seen.add(peer)
                    ports[peer], blobs[peer] = port, blob
                table = struct.pack(f"<{n_workers}I", *ports) + b"".join(blobs)
                for conn in conns:
                    conn.sendall(table)
            finally:
                for conn in conns:
                    conn.close()
    else:
        with _connect_retry((host, base_port), timeout, who) as conn:
            conn.settimeout(timeout)
            conn.sendall(_HELLO.pack(rank, data_port) + extra)
            raw = _recv_exact(conn, 4 * n_workers + width * n_workers, who)
        ports = list(struct.unpack(f"<{n_workers}I", raw[: 4 * n_workers]))
        rest = raw[4 * n_workers :]
        blobs = [rest[i * width : (i + 1) * width] for i in range(n_workers)]
    addresses = tuple((host, p) for p in ports)
    if payload is None:
        return addresses
    return addresses, blobs


# -------------------------------------------------------------------- session


class RingSession:
    """This rank's end of the NVLink group, reusable across collectives.

    Owns the native communicator (two IPC bucket slots + result buffer of
    ``capacity_bytes`` each, barrier flags, peer mappings) and a comm stream.
    Counters accumulate until ``close()``.
    """

    def __init__(
        self,
        config: WorkerConfig,
        comm: int,
        *,
        capacity_bytes: int = DEFAULT_CAPACITY_BYTES,
        timeout: float = _DEFAULT_TIMEOUT,
    ) -> None:
        import torch

        self.config = config
        self.counters = TransportCounters()
        self.capacity_bytes = int(capacity_bytes)
        self.device = torch.device("cuda", config.device_index)
        self._comm = comm
        self._timeout = timeout
        self.torch = torch
        self.stream = torch.cuda.Stream(device=self.device)
        self._staging = None
        self._tables: dict[tuple[int, int], _native.DeviceTable] = {}
        _native.call("mgw_comm_set_timeout_ms", comm, max(1, int(timeout * 1000)))

    @property
    def comm(self) -> int:
        if not self._comm:
            raise ProtocolError(f"rank {self.config.rank}: session is closed")
        return self._comm

    def close(self) -> None:
        for t in self._tables.values():
            t.close()
        self._tables.clear()
        if self._comm and getattr(self, "_local_group", False):
            return  # an in-process group is torn down as a whole by LocalGroup.close()
        if self._comm:
            # a peer's last pull kernel may still read this rank's slot after our last
            # collective returned: one zero-length collective (a barrier) before the region
            # is freed.  Best effort -- a dead or mismatched peer must not block close().
            try:
                _native.call("mgw_comm_set_timeout_ms", self._comm, 2000)
                _native.call("mgw_allreduce", self._comm, 0, _native.ALGO_ONESHOT, self.stream.cuda_stream)
                self.stream.synchronize()
            except Exception:
                pass
            _native.lib().mgw_comm_destroy(self._comm)
            self._comm = None

    def __enter__(self) -> "RingSession":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    # -- helpers used by the collectives
    def staging(self, n: int):
        torch = self.torch
        if self._staging is None or self._staging.numel() < n:
            self._staging = torch.empty(max(n, 1024), dtype=torch.float32, device=self.device)
        return self._staging

    def table(self, ptr: int, n: int) -> "_native.DeviceTable":
        key = (ptr, n)
        t = self._tables.get(key)
        if t is None:
            if len(self._tables) > 64:
                for old in self._tables.values():
                    old.close()
                self._tables.clear()
            t = _native.DeviceTable([(ptr, n, 0)])
            self._tables[key] = t
        return t

    def result_ptr(self) -> int:
        out = ctypes.c_void_p()
        _native.call("mgw_comm_result", self.comm, ctypes.byref(out))
        return out.value

    def raise_if_failed(self) -> None:
        code = ctypes.c_int()
        _native.call("mgw_comm_error", self.comm, ctypes.byref(code))
        if code.value == _native.DEV_OK:
            return
        who = f"rank {self.config.rank}"
        if code.value == _native.DEV_MISMATCH:
            raise ProtocolError(f"{who}: peers disagree on the collective (bucket length, algorithm, grid, dtype, "
                                "scale or group/iteration tag); buffer lengths likely disagree")
        if code.value == _native.DEV_TIMEOUT:
            raise ProtocolError(f"{who}: a peer never reached the collective within {self._timeout}s")
        raise ProtocolError(f"{who}: a peer aborted the collective")

    def clear_error(self) -> None:
        """Reset the device error word and this rank's abort flag after a ProtocolError
        (every rank, after a host-level barrier, before the next collective)."""
        _native.call("mgw_comm_clear_error", self.comm)

    def set_group_tag(self, layer_low: int, iteration: int = 0) -> None:
        """Tag the next collectives with (group, iteration), as the reference's frame header
        does (allreduce_net.py:340-345): ranks that disagree raise ProtocolError."""
        _native.call("mgw_comm_set_group_tag", self.comm, group_tag(layer_low, iteration))

    def account(self, n: int, algo: int, elem_bytes: int = 4) -> None:
        """NVLink payload accounting for one collective of n elements."""
        world, rank = self.config.n_workers, self.config.rank
        w = elem_bytes
        sizes, _ = _segments(n, world)
        c = self.counters
        c.frames_sent += 1
        c.frames_received += 1
        if algo == _native.ALGO_LL:  # pushed as 8-byte (epoch, payload) words: 2x the payload bytes
            c.rounds += 1
            c.payload_bytes_received += 2 * w * n * (world - 1)
            c.payload_bytes_sent += 2 * w * n * (world - 1)
        elif algo == _native.ALGO_LL128:  # the two-shot's bytes in 128-B lines of 120 B payload
            c.rounds += 2
            mine = sizes[rank]
            c.payload_bytes_received += w * ((world - 1) * mine + n - mine) * 16 // 15
            c.payload_bytes_sent += w * ((n - mine) + (world - 1) * mine) * 16 // 15
        elif algo == _native.ALGO_LL128_ONESHOT:  # (N-1) x M in 128-B lines of 120 B payload
            c.rounds += 1
            c.payload_bytes_received += w * n * (world - 1) * 16 // 15
            c.payload_bytes_sent += w * n * (world - 1) * 16 // 15
        elif algo in (_native.ALGO_ONESHOT, _native.ALGO_PUSH_ONESHOT):
            c.rounds += 1
            c.payload_bytes_received += w * n * (world - 1)
            c.payload_bytes_sent += w * n * (world - 1)
        else:
            c.rounds += 2
            mine = sizes[rank]
            c.payload_bytes_received += w * ((world - 1) * mine + n - mine)
            c.payload_bytes_sent += w * ((n - mine) + (world - 1) * mine)


def _segments(n_elements: int, n_parts: int) -> tuple[list[int], list[int]]:
    """Contiguous near-equal split; the first ``n % N`` parts get one extra element
    (allreduce_net.py:360-367).  Segment s starts the fold order of its elements."""
    q, r = divmod(n_elements, n_parts)
    sizes = [q + (1 if i < r else 0) for i in range(n_parts)]
    offsets = [0] * n_parts
    for i in range(1, n_parts):
        offsets[i] = offsets[i - 1] + sizes[i - 1]
    return sizes, offsets


LL_MAX_BYTES = 256 << 10  # push-based low-latency path (fused exchanges only), N >= 5


def ll_max_bytes(world: int) -> int:
    """AUTO's LL ceiling (mirrors mgw_comm_create): 1 MB at N = 2, 512 KB at N <= 4."""
    return (1 << 20) if world == 2 else ((512 << 10) if world <= 4 else LL_MAX_BYTES)


def group_tag(layer_low: int, iteration: int = 0) -> int:
    """32-bit group tag of (head layer, iteration) for mgw_comm_set_group_tag."""
    return ((int(iteration) * 0x9E3779B1) ^ int(layer_low)) & 0xFFFFFFFF


def _algo_for(session: RingSession, n: int, fused: bool = False, elem_bytes: int = 4) -> int:
    """The algorithm a collective of n elements runs under AUTO.  Fused exchanges ask the
    communicator itself (mgw_comm_pick_algo: thresholds set on it, NVLS, the push-row
    fallbacks); without a native communicator the host mirror ``_auto_rule`` answers."""
    comm = getattr(session, "_comm", None)
    if fused and comm:
        out = ctypes.c_int()
        _native.call("mgw_comm_pick_algo", comm, int(n), int(elem_bytes), ctypes.byref(out))
        return out.value
    return _auto_rule(session, n, fused)


def _auto_rule(session: RingSession, n: int, fused: bool = False) -> int:
    """Host mirror of pick_fused_algo / pick_algo at the default thresholds."""
    if fused:
        world = session.config.n_workers
        nbytes = 4 * n
        if world == 2 and (512 << 10) <= nbytes <= (16 << 20):
            return _native.ALGO_LL128_ONESHOT
        if 2 < world <= 4 and (256 << 10) <= nbytes <= (1 << 20):
            return _native.ALGO_LL128_ONESHOT
        if (1 << 20) <= nbytes <= ((128 << 20) if world == 2 else ((64 << 20) if world <= 4 else (16 << 20))):
            return _native.ALGO_LL128
        if 4 * n <= ll_max_bytes(world):
            return _native.ALGO_LL
        push_ok = 4 * n <= (1 << 30)
        if session.config.n_workers == 2:
            if 4 * n <= (16 << 20):
                return _native.ALGO_PUSH_ONESHOT
            return _native.ALGO_PUSH if push_ok else _native.ALGO_TWOSHOT
        if 4 * n <= (512 << 10):
            return _native.ALGO_PUSH_ONESHOT
        if 4 * n <= session_oneshot_max(session):
            return _native.ALGO_ONESHOT
        return _native.ALGO_PUSH if 4 * n >= (8 << 20) and push_ok else _native.ALGO_TWOSHOT
    return _native.ALGO_ONESHOT if 4 * n <= session_oneshot_max(session) else _native.ALGO_TWOSHOT


def session_oneshot_max(session: RingSession) -> int:
    world = session.config.n_workers
    return getattr(session, "oneshot_max_bytes", (8 << 20) // max(1, world - 1))


def set_oneshot_max(session: RingSession, nbytes: int) -> None:
    """Crossover between the pull one-shot and two-shot kernels (bytes) of the unfused
    path and of the fused AUTO choice at N >= 3 (at N = 2 the fused AUTO choice is the push
    one-shot up to 16 MB, see ``_algo_for``)."""
    _native.call("mgw_comm_set_oneshot_max", session.comm, int(nbytes))
    session.oneshot_max_bytes = int(nbytes)


def ring_allreduce(
    buffer: GradientBuffer,
    config: WorkerConfig,
    session: RingSession,
    *,
    iteration: int = 0,
) -> GradientBuffer:
    """Element-wise sum across all ranks, in place; returns ``buffer``.

    Collective.  Per element the sum is folded in the reference ring's order,
    so results are bit-identical to allreduce_net.py:370-411.  ``(layer_low,
    iteration)`` tag the collective as the reference's frame header does
    (allreduce_net.py:340-345): a rank issuing a different group or iteration raises
    ProtocolError on every rank instead of reducing unrelated buckets.
    """
    torch = session.torch
    values = buffer.values
    n = len(buffer)
    bf16 = _is_torch_tensor(values) and values.dtype == torch.bfloat16
    width = 2 if bf16 else 4
    if width * n > session.capacity_bytes:
        raise ValueError(f"buffer of {width * n} B exceeds the session capacity of {session.capacity_bytes} B")
    stream = session.stream
    numpy_payload = not _is_torch_tensor(values)
    with torch.cuda.device(session.device):
        if numpy_payload:
            dev = session.staging(n)
            if n:
                with torch.cuda.stream(stream):
                    dev[:n].copy_(torch.from_numpy(values))
            ptr = dev.data_ptr()
        else:
            if values.device != session.device:
                raise ValueError(f"tensor on {values.device}, session on {session.device}")
            stream.wait_stream(torch.cuda.current_stream(session.device))
            ptr = values.data_ptr()
        algo = _algo_for(session, n, fused=True, elem_bytes=width)
        handle = stream.cuda_stream
        session.set_group_tag(buffer.layer_low, iteration)
        if n and bf16:
            table = session.table(ptr, n)
            _native.call("mgw_allreduce_fused_bf16", session.comm, table.ptr, 1, n, ctypes.c_float(1.0),
                         _native.ALGO_AUTO, handle)
        elif n:
            # one kernel: pack -> all-reduce -> unpack, in place on the payload
            table = session.table(ptr, n)
            _native.call("mgw_allreduce_fused", session.comm, table.ptr, 1, n, ctypes.c_float(1.0),
                         _native.ALGO_AUTO, handle)
        else:
            # nothing to reduce, but still collective: a zero-length one-shot is a barrier
            algo = _native.ALGO_ONESHOT
            _native.call("mgw_allreduce", session.comm, 0, algo, handle)
        stream.synchronize()
        session.raise_if_failed()
        if numpy_payload and n:
            values[:] = session.staging(n)[:n].cpu().numpy()
    session.account(n, algo, width)
    return buffer


def bench_allreduce(
    sizes: list[int],
    config: WorkerConfig,
    session: RingSession,
    *,
    repeats: int = 5,
    warmups: int = 3,
) -> list[Measurement]:
    """Median device time of one group exchange (pack + all-reduce + unpack) per
    payload size (allreduce_net.py:414-445 semantics: sizes are positive multiples
    of 4 bytes; rank 0 returns the Measurements, other ranks an empty list).

    Each of the ``repeats`` samples is the mean of 8 back-to-back exchanges timed
    with one CUDA event pair on the comm stream (the kernel barrier keeps the ranks
    in lock-step), so neither host launch latency nor per-launch event cost enters
    the fit.  Every size is also checked once for the exact sum ``N(N+1)/2``.
    """
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    for nbytes in sizes:
        if not isinstance(nbytes, int) or nbytes <= 0 or nbytes % 4:
            raise ValueError(f"sizes must be positive multiples of 4 bytes, got {nbytes!r}")
        if nbytes > session.capacity_bytes:
            raise ValueError(f"size {nbytes} exceeds the session capacity of {session.capacity_bytes} B")
    torch = session.torch
    out: list[Measurement] = []
    world = config.n_workers
    handle = session.stream.cuda_stream
    loop = 8
    with torch.cuda.device(session.device), torch.cuda.stream(session.stream):
        for nbytes in sizes:
            n = nbytes // 4
            buf = torch.empty(n, dtype=torch.float32, device=session.device)
            table = _native.DeviceTable([(buf.data_ptr(), n, 0)])
            algo = _algo_for(session, n)
            times = []
            try:
                for r in range(repeats):
                    buf.fill_(float(config.rank + 1))
                    sec = ctypes.c_double()
                    _native.call("mgw_time_exchange", session.comm, table.ptr, 1, n, None, _native.ALGO_AUTO, 0,
                                 loop, warmups if r == 0 else 0, ctypes.byref(sec), handle)
                    times.append(sec.value)
                    session.account(n, algo)
                buf.fill_(float(config.rank + 1))
                _native.call("mgw_comm_pack", session.comm, table.ptr, 1, n, ctypes.c_float(1.0), handle)
                _native.call("mgw_allreduce", session.comm, n, algo, handle)
                _native.call("mgw_unpack", table.ptr, 1, session.result_ptr(), n, handle)
                session.stream.synchronize()
                session.raise_if_failed()
                if not bool((buf == float(world * (world + 1) // 2)).all()):
                    raise RuntimeError(f"rank {config.rank}: wrong all-reduce result at {nbytes} B")
            finally:
                table.close()
            if config.rank == 0:
                out.append(Measurement(nbytes=nbytes, seconds=statistics.median(times), n_nodes=world))
    return out


def run_emulation(
    profile: ModelProfile,
    plan: MergePlan | None,
    config: WorkerConfig,
    session: RingSession,
    iterations: int,
    *,
    warmup: int = 2,
    graph: bool = False,
    fused: bool = True,
    dtype=None,
) -> EmulationReport:
    """Measure the overlapped iteration (Algorithm 2) on the GPUs.

    Same contract as allreduce_net.py:463-578: arguments are validated before
    the session is touched; the gradients carry ``rank + 1 + layer % 5`` so the
    reduced values are exactly checkable; warm-up iterations run but are not
    reported.  Backward is simulated on a compute stream, each group's
    pack/all-reduce/unpack runs on the comm stream as soon as its head layer's
    gradient is ready.
    """
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if warmup < 0:
        raise ValueError("warmup must be >= 0")
    n_layers = profile.num_layers
    if plan is None:
        plan = MergePlan(frozenset(), n_layers)
    if plan.num_layers != n_layers:
        raise ValueError("plan does not match the profile's layer count")
    # element_bytes (2, 4 or 8, model_profile.py:24) only prices messages in the cost
    # model; the reference emulates every profile with fp32 buffers
    # (GradientBuffer.for_group, allreduce_net.py:98-120, :495-509), and so does this path.
    from .overlap import OverlappedIteration

    torch = session.torch
    # dtype=torch.bfloat16: the same Algorithm 2 on bf16 gradients (bf16 wire, fp32
    # accumulation); default fp32 as the reference
    width = 2 if dtype == torch.bfloat16 else 4
    largest = max((sum(p for _, p, _ in rows) for _, _, rows in _layout(profile, plan)), default=0)
    if width * largest > session.capacity_bytes:
        raise ValueError(f"largest group needs {width * largest} B, session capacity is {session.capacity_bytes} B")
    with torch.cuda.device(session.device):
        it = OverlappedIteration(
            profile,
            plan,
            comm=session.comm,
            rank=config.rank,
            world=config.n_workers,
            device=session.device,
            fill=True,
            graph=graph,
            fused=fused,
            dtype=dtype,
        )
        try:
            walls, computes, exposed = [], [], []
            per_group: dict[int, list[float]] = {low: [] for low, _, rows in it.layout if rows}
            verified = True
            count = 0
            for k in range(warmup + iterations):
                times = it.run()
                session.raise_if_failed()
                verified = it.verify() and verified
                count += it.sending_groups
                for (low, _, rows), t in zip(it.layout, times.group_comm):
                    if rows:
                        size = sum(p for _, p, _ in rows)
                        session.account(size, _algo_for(session, size, fused=fused, elem_bytes=width), width)
                        if k >= warmup:
                            per_group[low].append(t)
                if k >= warmup:
                    walls.append(times.t_iter)
                    computes.append(times.compute_time)
                    exposed.append(times.t_c_no)
            events = tuple(it.measured_timeline().events(profile))
        finally:
            it.close()
    return EmulationReport(
        rank=config.rank,
        n_workers=config.n_workers,
        iteration_seconds=tuple(walls),
        mean_seconds=statistics.fmean(walls),
        stddev_seconds=statistics.stdev(walls) if len(walls) > 1 else 0.0,
        group_comm_seconds={low: statistics.fmean(ts) for low, ts in per_group.items() if ts},
        verified=verified,
        allreduce_count=count,
        compute_seconds=tuple(computes),
        t_c_no_seconds=tuple(exposed),
        events=events,
    )


def _layout(profile, plan):
    from .overlap import group_layout

    return group_layout(profile, plan)


# ------------------------------------------------------------- process model


def _create_comm(rank: int, n_workers: int, device: int, capacity_bytes: int) -> tuple[int, bytes]:
    handle = ctypes.c_void_p()
    ipc = ctypes.create_string_buffer(_native.IPC_HANDLE_BYTES)
    _native.call("mgw_comm_create", rank, n_workers, device, int(capacity_bytes), ctypes.byref(handle), ipc)
    return handle.value, ipc.raw


def _pick_device(rank: int, n_workers: int, device: int | None) -> int:
    import torch

    visible = torch.cuda.device_count()
    if visible == 0:
        raise RuntimeError("no CUDA device visible: the B200 data path has no CPU fallback")
    if device is None:
        if visible < n_workers:
            raise RuntimeError(f"{n_workers} ranks need {n_workers} GPUs (one process per GPU); {visible} visible")
        device = rank
    if not 0 <= device < visible:
        raise ValueError(f"device {device} outside the {visible} visible GPUs")
    torch.cuda.set_device(device)
    return device


def open_ring(
    rank: int,
    n_workers: int,
    *,
    host: str = "127.0.0.1",
    base_port: int,
    chunk_elements: int = 1 << 22,
    timeout: float = _DEFAULT_TIMEOUT,
    capacity_bytes: int = DEFAULT_CAPACITY_BYTES,
    device: int | None = None,
) -> tuple[WorkerConfig, RingSession]:
    """Allocate this rank's IPC buckets, meet the others at ``base_port`` and
    map every peer's buckets (allreduce_net.py:581-605)."""
    dev = _pick_device(rank, n_workers, device)
    comm, ipc = _create_comm(rank, n_workers, dev, capacity_bytes)
    try:
        listener = socket.create_server((host, 0), backlog=2)
        try:
            data_port = listener.getsockname()[1]
            addresses, handles = rendezvous(rank, n_workers, host, base_port, data_port, timeout=timeout, payload=ipc)
        finally:
            listener.close()
        config = WorkerConfig(rank, n_workers, addresses, chunk_elements, device=dev)
        _native.call("mgw_comm_open_peers", comm, b"".join(handles))
        session = RingSession(config, comm, capacity_bytes=capacity_bytes, timeout=timeout)
    except BaseException:
        _native.lib().mgw_comm_destroy(comm)
        raise
    return config, session


class LocalGroup:
    """``n_workers`` ranks inside this process on ONE device (``mgw_comm_create_local``):
    every rank's communicator maps the others' regions directly and has its own session
    (settings, tags, error word).  ``allreduce_fused`` runs every rank's fused group
    exchange in ONE cooperative launch (``mgw_group_allreduce_fused``), so the real
    barrier / LL / push protocol -- and any disagreement between the ranks' settings --
    plays out between co-resident CTAs; kernels that wait on one another are never
    separate launches on one GPU.  Used by the single-GPU parity and protocol tests; the
    CTA cap is 2 * 148 / N so all ranks fit one launch.
    """

    def __init__(self, n_workers: int, *, device: int = 0, capacity_bytes: int = DEFAULT_CAPACITY_BYTES,
                 timeout: float = 10.0) -> None:
        import torch

        if not isinstance(n_workers, int) or not 2 <= n_workers <= _native.MAX_RANKS:
            raise ValueError(f"n_workers must lie in 2..{_native.MAX_RANKS}, got {n_workers!r}")
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device visible: the B200 data path has no CPU fallback")
        torch.cuda.set_device(device)
        self.torch = torch
        comms = (ctypes.c_void_p * n_workers)()
        _native.call("mgw_comm_create_local", n_workers, device, int(capacity_bytes), comms)
        self._comms = [comms[r] for r in range(n_workers)]
        addresses = tuple(("local", r) for r in range(n_workers))
        self.configs = [WorkerConfig(r, n_workers, addresses, device=device) for r in range(n_workers)]
        self.sessions = []
        for r in range(n_workers):
            sess = RingSession(self.configs[r], self._comms[r], capacity_bytes=capacity_bytes, timeout=timeout)
            sess._local_group = True
            self.sessions.append(sess)
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=device)

    @property
    def n_workers(self) -> int:
        return len(self.sessions)

    def allreduce_fused(self, rank_tensors, algo: int = _native.ALGO_AUTO, *, scales=None, absent=()) -> list:
        """In-place fused exchange of ``rank_tensors[r]`` (rank r's layer tensors in bucket
        order, all fp32 or all bf16) on every rank; returns each rank's ProtocolError or
        None.  Ranks listed in ``absent`` launch nothing (their peers time out)."""
        torch = self.torch
        world = self.n_workers
        bf16 = rank_tensors[0][0].dtype == torch.bfloat16
        tables, ns = [], []
        for r in range(world):
            rows, off = [], 0
            for t in rank_tensors[r]:
                rows.append((t.data_ptr(), t.numel(), off))
                off += t.numel()
            tables.append(_native.DeviceTable(rows))
            ns.append(-1 if r in absent else off)
        scales = [1.0] * world if scales is None else list(scales)
        try:
            self.stream.wait_stream(torch.cuda.current_stream())
            _native.call("mgw_group_allreduce_fused", (ctypes.c_void_p * world)(*self._comms),
                         (ctypes.c_void_p * world)(*[t.ptr for t in tables]), (ctypes.c_int64 * world)(*ns),
                         (ctypes.c_float * world)(*scales), world, int(algo), 2 if bf16 else 4,
                         self.stream.cuda_stream)
            self.stream.synchronize()
        finally:
            for t in tables:
                t.close()
        errors = []
        for r, sess in enumerate(self.sessions):
            if r in absent:
                errors.append(None)
                continue
            try:
                sess.raise_if_failed()
                errors.append(None)
            except ProtocolError as exc:
                errors.append(exc)
        return errors

    def bench_allreduce(self, sizes: list[int], *, repeats: int = 5, warmups: int = 3,
                        algo: int = _native.ALGO_AUTO) -> list[Measurement]:
        """``bench_allreduce`` (allreduce_net.py:414-445 semantics) for the in-process group:
        median device time of one fused group exchange per payload size, every rank's CTAs
        in one cooperative launch.  Each sample is 8 back-to-back group launches under one
        CUDA event pair, queued behind a short device spin so host launch latency stays out;
        every size is checked once for the exact sum N(N+1)/2."""
        if repeats < 1:
            raise ValueError("repeats must be >= 1")
        for nbytes in sizes:
            if not isinstance(nbytes, int) or nbytes <= 0 or nbytes % 4:
                raise ValueError(f"sizes must be positive multiples of 4 bytes, got {nbytes!r}")
            if nbytes > self.sessions[0].capacity_bytes:
                raise ValueError(f"size {nbytes} exceeds the session capacity of {self.sessions[0].capacity_bytes} B")
        torch = self.torch
        world = self.n_workers
        out: list[Measurement] = []
        loop = 8
        for nbytes in sizes:
            n = nbytes // 4
            bufs = [torch.empty(n, dtype=torch.float32, device=self.device) for _ in range(world)]
            tables = [_native.DeviceTable([(b.data_ptr(), n, 0)]) for b in bufs]
            args = ((ctypes.c_void_p * world)(*self._comms), (ctypes.c_void_p * world)(*[t.ptr for t in tables]),
                    (ctypes.c_int64 * world)(*([n] * world)), (ctypes.c_float * world)(*([1.0] * world)), world,
                    int(algo), 4, self.stream.cuda_stream)
            try:
                self.stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(self.stream):
                    for _ in range(warmups):
                        _native.call("mgw_group_allreduce_fused", *args)
                    times = []
                    for _ in range(repeats):
                        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        _native.call("mgw_spin_ns", 2_000_000, self.stream.cuda_stream)
                        start.record(self.stream)
                        for _ in range(loop):
                            _native.call("mgw_group_allreduce_fused", *args)
                        end.record(self.stream)
                        end.synchronize()
                        times.append(start.elapsed_time(end) * 1e-3 / loop)
                    for r, b in enumerate(bufs):
                        b.fill_(float(r + 1))
                    _native.call("mgw_group_allreduce_fused", *args)
                    self.stream.synchronize()
                for sess in self.sessions:
                    sess.raise_if_failed()
                for b in bufs:
                    if not bool((b == float(world * (world + 1) // 2)).all()):
                        raise RuntimeError(f"wrong all-reduce result at {nbytes} B")
            finally:
                for t in tables:
                    t.close()
            out.append(Measurement(nbytes=nbytes, seconds=statistics.median(times), n_nodes=world))
        return out

    def clear_errors(self) -> None:
        for sess in self.sessions:
            sess.clear_error()

    def close(self) -> None:
        for sess in self.sessions:
            for t in sess._tables.values():
                t.close()
            sess._tables.clear()
        if self._comms:
            self.stream.synchronize()
            for c in self._comms:
                _native.lib().mgw_comm_destroy(c)
            for sess in self.sessions:
                sess._comm = None
            self._comms = []

    def __enter__(self) -> "LocalGroup":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def exchange_handles_dist(handle: bytes, *, group=None) -> bytes:
    """All-gather every rank's 64-byte IPC handle through torch.distributed; returns the
    rank-ordered concatenation ``mgw_comm_open_peers`` expects."""
    import torch.distributed as dist

    if len(handle) != _native.IPC_HANDLE_BYTES:
        raise ValueError(f"IPC handles are {_native.IPC_HANDLE_BYTES} bytes, got {len(handle)}")
    handles: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, bytes(handle), group=group)
    if any(h is None or len(h) != _native.IPC_HANDLE_BYTES for h in handles):
        raise ProtocolError("a rank contributed a malformed IPC handle")
    return b"".join(handles)


def open_session_dist(
    *,
    capacity_bytes: int = DEFAULT_CAPACITY_BYTES,
    timeout: float = _DEFAULT_TIMEOUT,
    group=None,
) -> tuple[WorkerConfig, RingSession]:
    """``open_ring`` for processes launched by torchrun: the IPC handles travel
    through an initialised ``torch.distributed`` group instead of the TCP
    rendezvous (device = LOCAL_RANK)."""
    import os

    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    comm, ipc = _create_comm(rank, world, dev, capacity_bytes)
    try:
        _native.call("mgw_comm_open_peers", comm, exchange_handles_dist(ipc, group=group))
        addresses = tuple(("torch.distributed", r) for r in range(world))
        config = WorkerConfig(rank, world, addresses, device=dev)
        session = RingSession(config, comm, capacity_bytes=capacity_bytes, timeout=timeout)
    except BaseException:
        _native.lib().mgw_comm_destroy(comm)
        raise
    return config, session


def enable_nvls(session: RingSession, nbytes: int, *, min_bytes: int = 0, group=None) -> None:
    """Opt-in NVSwitch multicast (NVLS) exchange on a torchrun-launched session.

    Rank 0 creates a multicast object of ``nbytes`` and hands its POSIX fd to every
    other rank over an abstract Unix socket (SCM_RIGHTS); every rank adds its device,
    then binds and maps its copy.  Afterwards ``MGW_ALGO_NVLS`` (or AUTO for buckets
    >= ``min_bytes`` when non-zero) reduces in the switch.  NVLS sums in the switch's
    order: identical on every rank and within fp32 rounding of the exact sum, but not
    bit-identical to the reference ring -- so it is never on by default.
    """
    import os
    import secrets

    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ok = ctypes.c_int()
    _native.call("mgw_nvls_supported", session.config.device_index, ctypes.byref(ok))
    flags: list = [None] * world
    dist.all_gather_object(flags, bool(ok.value), group=group)
    if not all(flags):
        raise RuntimeError("NVLS (CUDA multicast) is not supported on every device of the group")
    box = [secrets.token_hex(8) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    name = "\0mgwfbp-nvls-" + box[0]
    comm = session.comm
    if rank == 0:
        fd = ctypes.c_int(-1)
        _native.call("mgw_nvls_create", comm, int(nbytes), ctypes.byref(fd))
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(world)
        dist.barrier(group=group)
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"f"], [fd.value])
        finally:
            srv.close()
            os.close(fd.value)
    else:
        dist.barrier(group=group)
        with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as s:
            s.connect(name)
            _, fds, _, _ = socket.recv_fds(s, 1, 1)
        try:
            _native.call("mgw_nvls_import", comm, fds[0], int(nbytes))
        finally:
            os.close(fds[0])
    _native.call("mgw_nvls_add_device", comm)
    dist.barrier(group=group)
    _native.call("mgw_nvls_bind", comm)
    dist.barrier(group=group)
    if min_bytes:
        _native.call("mgw_comm_set_nvls_min", comm, int(min_bytes))
    session.nvls_bytes = int(nbytes)


def _worker_main(result_q, rank, n_workers, host, base_port, chunk_elements, timeout, capacity_bytes, task) -> None:
    try:
        config, session = open_ring(
            rank,
            n_workers,
            host=host,
            base_port=base_port,
            chunk_elements=chunk_elements,
            timeout=timeout,
            capacity_bytes=capacity_bytes,
        )
        try:
            value = task(config, session)
        finally:
            session.close()
        result_q.put((rank, None, value))
    except BaseException:
        result_q.put((rank, traceback.format_exc(), None))


def run_workers(
    n_workers: int,
    task,
    *,
    host: str = "127.0.0.1",
    base_port: int | None = None,
    chunk_elements: int = 1 << 22,
    timeout: float = 120.0,
    capacity_bytes: int = DEFAULT_CAPACITY_BYTES,
):
    """Spawn one process per rank (one GPU each), open the group in every
    process and run ``task(config, session)`` collectively; returns
    ``{rank: result}`` or raises RuntimeError with the failed tracebacks
    (allreduce_net.py:622-683)."""
    if n_workers < 2:
        raise ValueError("n_workers must be >= 2")
    if base_port is None:
        base_port = _free_port(host)
    ctx = get_context("spawn")
    result_q = ctx.Queue()
    procs = [
        ctx.Process(
            target=_worker_main,
            args=(result_q, rank, n_workers, host, base_port, chunk_elements, timeout, capacity_bytes, task),
            daemon=True,
        )
        for rank in range(n_workers)
    ]
    for p in procs:
        p.start()
    results: dict[int, object] = {}
    errors: list[tuple[int, str]] = []
    deadline = time.monotonic() + timeout
    try:
        while len(results) + len(errors) < n_workers and time.monotonic() < deadline:
            try:
                rank, err, value = result_q.get(timeout=0.25)
            except queue.Empty:
                if any(p.exitcode not in (None, 0) for p in procs):
                    break
                continue
            if err is None:
                results[rank] = value
            else:
                errors.append((rank, err))
    finally:
        for p in procs:
            p.join(timeout=10.0)
        for p in procs:
            if p.is_alive():
                p.terminate()
                p.join(timeout=5.0)
    if errors:
        detail = "\n".join(f"--- worker {rank} ---\n{err}" for rank, err in sorted(errors))
        raise RuntimeError(f"{len(errors)} of {n_workers} workers failed:\n{detail}")
    if len(results) < n_workers:
        missing = sorted(set(range(n_workers)) - set(results))
        raise RuntimeError(f"workers {missing} never reported (crash or timeout)")
    return results


def _bench_task(config: WorkerConfig, session: RingSession, *, sizes, repeats, warmups):
    return bench_allreduce(list(sizes), config, session, repeats=repeats, warmups=warmups)


def _emulation_task(config: WorkerConfig, session: RingSession, *, profile, plan, iterations, warmup, graph=False):
    return run_emulation(profile, plan, config, session, iterations, warmup=warmup, graph=graph)


def bench_local(
    n_workers: int,
    sizes: list[int],
    *,
    repeats: int = 5,
    warmups: int = 3,
    host: str = "127.0.0.1",
    base_port: int | None = None,
    timeout: float = 120.0,
) -> list[Measurement]:
    """Spawn the group on this box's GPUs and time the given payload sizes."""
    for nbytes in sizes:
        if not isinstance(nbytes, int) or nbytes <= 0 or nbytes % 4:
            raise ValueError(f"sizes must be positive multiples of 4 bytes, got {nbytes!r}")
    capacity = max(max(sizes), 1 << 20)
    results = run_workers(
        n_workers,
        partial(_bench_task, sizes=tuple(sizes), repeats=repeats, warmups=warmups),
        host=host,
        base_port=base_port,
        timeout=timeout,
        capacity_bytes=capacity,
    )
    return results[0]


def emulate_local(
    n_workers: int,
    profile: ModelProfile,
    plan: MergePlan | None,
    iterations: int,
    *,
    warmup: int = 2,
    host: str = "127.0.0.1",
    base_port: int | None = None,
    timeout: float = 300.0,
    graph: bool = False,
) -> dict[int, EmulationReport]:
    """Spawn the group on this box's GPUs and measure the emulated iteration."""
    if plan is None:
        plan = MergePlan(frozenset(), profile.num_layers)
    largest = max((sum(p for _, p, _ in rows) for _, _, rows in _layout(profile, plan)), default=0)
    results = run_workers(
        n_workers,
        partial(_emulation_task, profile=profile, plan=plan, iterations=iterations, warmup=warmup, graph=graph),
        host=host,
        base_port=base_port,
        timeout=timeout,
        capacity_bytes=max(4 * largest, 1 << 20),
    )
    return {rank: report for rank, report in results.items()}
