"""Algorithm 2 on CUDA streams: simulated backward overlapped with merged all-reduces.

The reference emulates one training iteration with a compute thread that burns
``t_f`` and each ``t_b`` (``_delay``) and pushes ready layers onto a queue, and a
main thread that packs each layer and fires the group's ring all-reduce when
the group's lowest layer arrives (``/root/reference/pkg/src/mgwfbp/
allreduce_net.py:463-578``).  Here the same iteration is a native schedule
(``mgw_sched_*`` in the C ABI):

* compute stream -- a clock-mark kernel, then per merge group (send order) an
  optional gradient "production" kernel (``MGW_SCHED_FILL``: writes the
  reference's ``rank + 1 + layer % 5`` pattern) and a deadline spin until the
  group head's readiness ``tau_b[head] + t_b[head]``; deadlines are absolute
  from the iteration start, so launch gaps never accumulate into compute time;
* comm stream -- per group: wait for the head's event, K1 pack(+scale) into
  the IPC bucket, K2/K3 all-reduce over NVLink, K4 unpack; one stream is the
  simulator's single serialized channel (``schedule_sim.py:7-13``);
* timing -- CUDA events: iteration start, backward end, comm end, and every
  group's comm span, which give ``t_iter``, ``compute_time`` and
  ``t_c_no = t_iter - compute_time`` exactly as ``Timeline`` defines them.

With ``graph=True`` the whole iteration is captured once and replayed as one
CUDA graph launch; the collectives take their epochs from a device counter so
replays stay correctly synchronised.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

from . import _native
from .merge_planner import MergePlan
from .model_profile import ModelProfile
from .schedule_sim import backward_start_times

__all__ = ["IterationTimes", "OverlappedIteration", "group_layout"]


@dataclass(frozen=True)
class IterationTimes:
    t_iter: float
    compute_time: float
    group_comm: tuple[float, ...]  # send order

    @property
    def t_c_no(self) -> float:
        return self.t_iter - self.compute_time


def group_layout(profile: ModelProfile, plan: MergePlan):
    """Send-ordered groups with their bucket rows.

    Returns ``[(low, high, [(layer, params, bucket_offset), ...]), ...]``,
    descending by layer; within a group layer ``high`` sits at offset 0 and the
    rest follow downward (allreduce_net.py:499-509).  Silent layers get no row.
    """
    counts = profile.param_counts()
    out = []
    for low, high in reversed(plan.groups()):
        rows, off = [], 0
        for layer in range(high, low - 1, -1):
            p = counts[layer - 1]
            if p:
                rows.append((layer, p, off))
                off += p
        out.append((low, high, rows))
    return out


class OverlappedIteration:
    """One rank's emulated iteration, ready to run repeatedly.

    ``comm`` is a native communicator handle (``None`` for a single GPU, where
    the iteration packs/unpacks but exchanges nothing).  ``tensors`` maps layer
    index -> a CUDA float32 tensor of that layer's gradient; created here when
    omitted.  ``fill`` selects per-iteration gradient production with the
    reference pattern; ``host_io`` adds the end-to-end H2D/D2H legs.  ``fused`` runs one
    kernel per group (N = 1: the single-rank group kernel); ``pdl`` launches each group's
    exchange while its gradient fill still runs (programmatic dependent launch).
    """

    def __init__(
        self,
        profile: ModelProfile,
        plan: MergePlan | None,
        *,
        comm: int | None,
        rank: int,
        world: int,
        device,
        scale: float = 1.0,
        fill: bool = True,
        graph: bool = False,
        host_io: bool = False,
        algo: int = _native.ALGO_AUTO,
        tensors: dict | None = None,
        fused: bool = False,
        pdl: bool = True,
        dtype=None,
    ) -> None:
        import torch

        # element_bytes (2, 4, 8) only prices messages in the cost model: the emulation
        # moves fp32 buffers for every profile, as the reference does (allreduce_net.py:495-509)
        if plan is None:
            plan = MergePlan(frozenset(), profile.num_layers)
        if plan.num_layers != profile.num_layers:
            raise ValueError("plan does not match the profile's layer count")
        self.profile, self.plan = profile, plan
        self.rank, self.world = rank, world
        self.device = torch.device(device)
        if host_io:
            fill = False  # gradients arrive from the host instead
        self.fill, self.host_io, self.scale = fill, host_io, float(scale)
        self.torch = torch
        self.dtype = torch.float32 if dtype is None else dtype
        if self.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError(f"gradients are fp32 or bf16, got {self.dtype}")
        self.bf16 = self.dtype == torch.bfloat16
        if self.bf16 and host_io:
            raise ValueError("the end-to-end host legs move fp32 buffers")
        counts = profile.param_counts()
        if tensors is None:
            tensors = {
                layer: torch.zeros(p, dtype=self.dtype, device=self.device)
                for layer, p in enumerate(counts, start=1)
                if p
            }
        self.tensors = tensors
        t_b = profile.backward_times()
        tau_b = backward_start_times(profile)
        self.layout = group_layout(profile, plan)

        rows, fills, groups = [], [], []
        self.host_src, self.host_dst = {}, {}
        for low, high, grows in self.layout:
            begin = len(rows)
            n_elem = 0
            for layer, p, off in grows:
                t = tensors[layer]
                if t.numel() != p or t.dtype != self.dtype or not t.is_contiguous():
                    raise ValueError(f"layer {layer}: need a contiguous {self.dtype} tensor of {p} elements")
                rows.append((t.data_ptr(), p, off))
                fills.append(float(rank + 1 + layer % 5))
                n_elem += p
            ready = tau_b[low - 1] + t_b[low - 1]
            g = _native.Group()
            g.head_layer, g.desc_begin, g.desc_count = low, begin, len(rows) - begin
            g.algo, g.n_elem, g.ready_ns = algo, n_elem, int(round(ready * 1e9))
            groups.append(g)
        self.n_groups = len(groups)
        self.sending_groups = sum(1 for g in groups if g.n_elem)
        desc = _native.desc_array(rows)
        garr = (_native.Group * len(groups))(*groups)
        fill_arr = (ctypes.c_float * max(1, len(fills)))(*fills) if fill else None
        flags = (_native.SCHED_FILL if fill else 0) | (_native.SCHED_GRAPH if graph else 0)
        if fused:
            flags |= _native.SCHED_FUSED
        if self.bf16:
            flags |= _native.SCHED_BF16  # bf16 wire and bucket, fp32 accumulation (always fused)
        if pdl and fill:
            flags |= _native.SCHED_PDL  # the exchange launches while the fill runs
        self.fused = fused
        src_arr = dst_arr = None
        if host_io:
            flags |= _native.SCHED_HOSTIO
            src_ptrs, dst_ptrs = [], []
            for low, high, grows in self.layout:
                for layer, p, off in grows:
                    hs = torch.empty(p, dtype=torch.float32).pin_memory()
                    hs.fill_(float(rank + 1 + layer % 5))
                    hd = torch.empty(p, dtype=torch.float32).pin_memory()
                    self.host_src[layer], self.host_dst[layer] = hs, hd
                    src_ptrs.append(hs.data_ptr())
                    dst_ptrs.append(hd.data_ptr())
            src_arr = (ctypes.c_void_p * max(1, len(src_ptrs)))(*src_ptrs)
            dst_arr = (ctypes.c_void_p * max(1, len(dst_ptrs)))(*dst_ptrs)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.call(
                "mgw_sched_create",
                comm,
                desc,
                len(rows),
                garr,
                len(groups),
                ctypes.c_float(self.scale),
                flags,
                fill_arr,
                src_arr,
                dst_arr,
                ctypes.byref(handle),
            )
        self._sched = handle.value
        self.n_rows = len(rows)
        self.compute_stream = torch.cuda.Stream(device=self.device)
        # high priority: a ready group's exchange is scheduled ahead of queued compute CTAs
        self.comm_stream = torch.cuda.Stream(device=self.device, priority=-1)
        n = ctypes.c_int()
        _native.call("mgw_sched_launches", self._sched, ctypes.byref(n))
        self.launches_per_iteration = n.value
        # verification table: every layer once, global offsets
        self._check_rows, self._expect = [], []
        off = 0
        for low, high, grows in self.layout:
            for layer, p, _ in grows:
                self._check_rows.append((tensors[layer].data_ptr(), p, off))
                self._expect.append(self._expected(layer))
                off += p
        self._check_table = None
        self._expect_dev = None

    def _expected(self, layer: int) -> float:
        n = self.world
        return float(n * (n + 1) // 2 + n * (layer % 5)) * self.scale if self.world > 1 else float(1 + layer % 5) * self.scale

    def run(self) -> IterationTimes:
        """Enqueue one iteration and wait for its timings."""
        _native.call("mgw_sched_run", self._sched, self.compute_stream.cuda_stream, self.comm_stream.cuda_stream)
        return self.times()

    def launch(self) -> None:
        _native.call("mgw_sched_run", self._sched, self.compute_stream.cuda_stream, self.comm_stream.cuda_stream)

    def times(self) -> IterationTimes:
        t_iter, compute = ctypes.c_double(), ctypes.c_double()
        groups = (ctypes.c_double * max(1, self.n_groups))()
        _native.call("mgw_sched_times", self._sched, ctypes.byref(t_iter), ctypes.byref(compute), groups)
        return IterationTimes(t_iter.value, compute.value, tuple(groups[: self.n_groups]))

    def kernel_times(self) -> tuple[tuple[float, ...], tuple[float, ...], tuple[float, ...]]:
        """Per-group (pack, all-reduce, unpack) device seconds of the last iteration."""
        k = max(1, self.n_groups)
        pack, ar, unpack = (ctypes.c_double * k)(), (ctypes.c_double * k)(), (ctypes.c_double * k)()
        _native.call("mgw_sched_kernel_times", self._sched, pack, ar, unpack)
        g = self.n_groups
        return tuple(pack[:g]), tuple(ar[:g]), tuple(unpack[:g])

    def measured_timeline(self, strategy=None):
        """The last iteration as a ``Timeline`` (schedule_sim.py:65-100), from the kernels'
        own %globaltimer stamps relative to the iteration's clock mark (the simulated
        backward's origin): a group's backward is shifted by how late its gradient fill
        ended against the schedule, its head layer's comm row is the measured exchange
        window (first kernel entry .. last exit), merged layers carry zero-length rows as
        in the simulator, and t_iter = the later of the last exchange and the backward.
        ``Timeline.events(profile)`` then gives the measured Gantt rows."""
        from .schedule_sim import OverlapCase, Strategy, Timeline

        k = max(1, self.n_groups)
        ready, c0, c1 = (ctypes.c_double * k)(), (ctypes.c_double * k)(), (ctypes.c_double * k)()
        _native.call("mgw_sched_events", self._sched, ready, c0, c1)
        prof = self.profile
        n = prof.num_layers
        t_b = prof.backward_times()
        tau_sim = backward_start_times(prof)
        tau_b, tau_c, t_c, comm_end = list(tau_sim), [0.0] * n, [0.0] * n, [0.0] * n
        for g, (low, high, grows) in enumerate(self.layout):
            due = tau_sim[low - 1] + t_b[low - 1]
            late = ready[g] - due if ready[g] >= 0.0 else 0.0
            for layer in range(low, high + 1):
                tau_b[layer - 1] = tau_sim[layer - 1] + late
            start, end = (c0[g], c1[g]) if (grows and c0[g] >= 0.0) else (due + late, due + late)
            for layer in range(low, high + 1):
                tau_c[layer - 1] = comm_end[layer - 1] = start
            tau_c[low - 1], comm_end[low - 1], t_c[low - 1] = start, end, end - start
        compute = tau_b[0] + t_b[0]
        t_iter = max([compute] + comm_end)
        return Timeline(strategy=strategy or Strategy.MGWFBP, tau_b=tuple(tau_b), tau_c=tuple(tau_c),
                        t_c=tuple(t_c), comm_end=tuple(comm_end), t_iter=t_iter, compute_time=compute,
                        t_c_no=t_iter - compute, case=OverlapCase.NOT_APPLICABLE)

    def group_bytes(self) -> tuple[int, ...]:
        """Bucket bytes of each group, send order."""
        width = 2 if self.bf16 else 4
        return tuple(width * sum(p for _, p, _ in rows) for _, _, rows in self.layout)

    def verify(self) -> bool:
        """Every layer equals the reference's expected reduced constant
        (allreduce_net.py:507, ``N(N+1)/2 + N(layer % 5)``)."""
        torch = self.torch
        if not self._check_rows:
            return True
        if self.bf16:  # the expected sums are small integers, exact in bf16
            self.compute_stream.synchronize()
            self.comm_stream.synchronize()
            return all(bool((self.tensors[layer] == self._expected(layer)).all())
                       for _, _, grows in self.layout for layer, _, _ in grows)
        if self._check_table is None:
            self._check_table = _native.DeviceTable(self._check_rows)
            self._expect_dev = torch.tensor(self._expect, dtype=torch.float32, device=self.device)
        bad = ctypes.c_int64()
        self.compute_stream.synchronize()
        self.comm_stream.synchronize()
        _native.call(
            "mgw_check_const",
            self._check_table.ptr,
            self._check_table.n,
            self._expect_dev.data_ptr(),
            ctypes.byref(bad),
            self.comm_stream.cuda_stream,
        )
        if self.host_io:
            for low, high, grows in self.layout:
                for layer, p, _ in grows:
                    if not bool((self.host_dst[layer] == self._expected(layer)).all()):
                        return False
        return bad.value == 0

    def io_bytes(self) -> tuple[int, int]:
        total = 4 * sum(p for _, _, grows in self.layout for _, p, _ in grows)
        return (total, total) if self.host_io else (0, 0)

    def close(self) -> None:
        if getattr(self, "_sched", None):
            _native.lib().mgw_sched_destroy(self._sched)
            self._sched = None
        if getattr(self, "_check_table", None) is not None:
            self._check_table.close()
            self._check_table = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def mean_and_stdev(xs) -> tuple[float, float]:
    xs = list(xs)
    mean = math.fsum(xs) / len(xs)
    if len(xs) < 2:
        return mean, 0.0
    var = math.fsum((x - mean) ** 2 for x in xs) / (len(xs) - 1)
    return mean, math.sqrt(var)
