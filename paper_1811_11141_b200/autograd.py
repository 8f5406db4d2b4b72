"""MG-WFBP on a real backward pass: merged all-reduce driven by autograd gradient readiness.

The reference emulates backward with timed delays (``allreduce_net.py:516-529``);
SURVEY §8(f)-2 names the real thing as the next step: a parameter's gradient is
"ready" when autograd has accumulated it (``register_post_accumulate_grad_hook``).
``MergedGradientSync`` attaches to a model's parameters (the "layers", in forward
order, one per tensor as in ``bert_base_like``), counts readiness per merge group, and
as soon as a group is complete launches its fused pack -> all-reduce -> unpack kernel
(``mgw_allreduce_fused``) on a comm stream that waits on an event recorded on the
backward stream -- Algorithm 2 with real compute.  ``finish()`` makes the current
stream wait for the comm stream before the optimizer step.

``measure_profile`` times a real backward with per-parameter events and returns a
``ModelProfile`` (the reference's layer-profile format, ``model_profile.py:27-97``)
that ``find_merge_plan`` consumes unchanged.

All ranks launch their group collectives in the same order because autograd's
execution order is deterministic for identical graphs; groups are counted, not
assumed to finish in strictly descending layer order.
"""

from __future__ import annotations

import ctypes
from functools import partial

from . import _native
from .merge_planner import MergePlan
from .model_profile import LayerProfile, ModelProfile

__all__ = ["MergedGradientSync", "measure_profile", "trainable_parameters"]


def trainable_parameters(model) -> list:
    """Parameters in registration (forward) order that receive gradients."""
    return [p for p in model.parameters() if p.requires_grad]


class MergedGradientSync:
    """Merged-gradient all-reduce hooked into autograd (one process per GPU).

    ``comm`` is a native communicator (``RingSession.comm``) or None for a single GPU
    (then only the optional ``scale`` is applied).  ``plan`` groups the parameter list
    (layer k = params[k-1]); the group's bucket layout is the reference's (highest
    layer first).  ``scale=1/N`` averages.  ``priority`` is the comm stream's CUDA
    priority (-1 = high); ``gate`` launches each collective only once every peer has
    reached it (``mgw_comm_set_gate``).
    """

    def __init__(self, params, plan: MergePlan, *, comm=None, world: int = 1, scale: float = 1.0,
                 algo: int = _native.ALGO_AUTO, sync_after_backward: bool = False, max_ctas: int | None = None,
                 priority: int = 0, gate: bool = False):
        import torch

        self.torch = torch
        self.params = list(params)
        if plan.num_layers != len(self.params):
            raise ValueError(f"plan covers {plan.num_layers} layers, model has {len(self.params)} trainable tensors")
        for p in self.params:
            if p.dtype not in (torch.float32, torch.bfloat16):
                raise ValueError("the B200 data path reduces fp32 or bf16 gradients")
        self.plan = plan
        self.comm, self.world, self.scale, self.algo = comm, world, float(scale), algo
        self.sync_after_backward = sync_after_backward
        if max_ctas is not None and comm is not None:
            # overlapped collectives share the SMs with backward: bound their CTA budget
            _native.call("mgw_comm_set_max_ctas", comm, int(max_ctas))
        if comm is not None:
            # gate: every bulk kernel waits (one warp) until all peers reached it
            _native.call("mgw_comm_set_gate", comm, int(gate))
        self.groups = plan.groups()  # ascending (low, high)
        self.group_of = {}
        for gid, (low, high) in enumerate(self.groups):
            for layer in range(low, high + 1):
                self.group_of[layer] = gid
        self.size = [high - low + 1 for low, high in self.groups]
        # bf16 groups: bf16 on the wire, fp32 accumulation (mgw_group_launch_bf16)
        self.bf16 = []
        for low, high in self.groups:
            kinds = {self.params[layer - 1].dtype for layer in range(low, high + 1)}
            if len(kinds) != 1:
                raise ValueError(f"group {(low, high)} mixes gradient dtypes {sorted(map(str, kinds))}")
            self.bf16.append(kinds == {torch.bfloat16})
        self.count = [0] * len(self.groups)
        self.tables: dict[int, tuple] = {}
        self.events: dict[int, int] = {}
        # priority < 0 puts the comm stream ahead of backward in the CTA scheduler, so a
        # ready group's collective is not queued behind a wave of backward blocks
        self.stream = torch.cuda.Stream(priority=priority)
        self.launched = 0
        self.pending: list[int] = []
        self.handles = [p.register_post_accumulate_grad_hook(partial(self._ready, k))
                        for k, p in enumerate(self.params, start=1)]

    def _table(self, gid):
        low, high = self.groups[gid]
        grads = [self.params[layer - 1].grad for layer in range(high, low - 1, -1)]
        key = tuple(g.data_ptr() for g in grads)
        cached = self.tables.get(gid)
        if cached is None or cached[0] != key:
            if cached is not None:
                cached[1].close()
            rows, off = [], 0
            for g in grads:
                if not g.is_contiguous():
                    raise ValueError("gradients must be contiguous")
                rows.append((g.data_ptr(), g.numel(), off))
                off += g.numel()
            cached = (key, _native.DeviceTable(rows), off)
            self.tables[gid] = cached
        return cached[1], cached[2]

    def _event(self, gid):
        ev = self.events.get(gid)
        if ev is None:
            handle = ctypes.c_void_p()
            _native.call("mgw_event_create", ctypes.byref(handle))
            ev = self.events[gid] = handle.value
        return ev

    def _launch(self, gid):
        torch = self.torch
        table, n = self._table(gid)
        if self.comm is not None and self.world > 1:
            # one native call: event on the backward (current) stream -> comm stream waits
            # -> fused pack / all-reduce / unpack of the group
            fn = "mgw_group_launch_bf16" if self.bf16[gid] else "mgw_group_launch"
            _native.call(fn, self.comm, table.ptr, table.n, n, ctypes.c_float(self.scale), self.algo,
                         torch.cuda.current_stream().cuda_stream, self.stream.cuda_stream, self._event(gid))
        elif self.scale != 1.0:
            ev = torch.cuda.Event()
            ev.record()
            self.stream.wait_event(ev)
            with torch.cuda.stream(self.stream):
                for layer in range(self.groups[gid][0], self.groups[gid][1] + 1):
                    self.params[layer - 1].grad.mul_(self.scale)
        self.launched += 1

    def _ready(self, layer, param):
        gid = self.group_of[layer]
        self.count[gid] += 1
        if self.count[gid] == self.size[gid]:
            if self.sync_after_backward:
                self.pending.append(gid)  # SyncEASGD-style: everything after backward
            else:
                self._launch(gid)

    def finish(self):
        """Call after ``loss.backward()``: the optimizer's stream waits for every group."""
        for gid in self.pending:
            self._launch(gid)
        self.pending.clear()
        if any(c != s for c, s in zip(self.count, self.size)):
            missing = [g for g, (c, s) in enumerate(zip(self.count, self.size)) if c != s]
            raise RuntimeError(f"groups {missing[:5]} never completed: a parameter got no gradient")
        self.count = [0] * len(self.groups)
        self.torch.cuda.current_stream().wait_stream(self.stream)

    def close(self):
        for h in self.handles:
            h.remove()
        for _, table, _ in self.tables.values():
            table.close()
        self.tables.clear()
        for ev in self.events.values():
            _native.lib().mgw_event_destroy(ev)
        self.events.clear()


def measure_profile(model, step, *, name="measured", repeats=5) -> ModelProfile:
    """Per-parameter backward timing of a real model.

    ``step()`` runs forward + loss and returns the loss (it is called with gradients
    enabled).  Each parameter's post-accumulate hook records a CUDA event; layer k's
    backward time is the gap between the event of the parameter before it in readiness
    order and its own; ``forward_time`` is the forward span.  Medians over ``repeats``.
    """
    import statistics

    import torch

    params = trainable_parameters(model)
    n = len(params)
    samples_tb = [[] for _ in range(n)]
    samples_tf = []
    for _ in range(repeats + 1):
        events = {}
        handles = []

        def hook(k, p):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events[k] = ev

        for k, p in enumerate(params):
            handles.append(p.register_post_accumulate_grad_hook(partial(hook, k)))
        start, mid = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        model.zero_grad(set_to_none=False)
        start.record()
        loss = step()
        mid.record()
        loss.backward()
        torch.cuda.synchronize()
        for h in handles:
            h.remove()
        if len(events) != n:
            raise RuntimeError("some parameters received no gradient")
        order = sorted(range(n), key=lambda k: start.elapsed_time(events[k]))
        prev = mid
        times = {}
        for k in order:
            times[k] = max(0.0, prev.elapsed_time(events[k]) * 1e-3)
            prev = events[k]
        samples_tf.append(start.elapsed_time(mid) * 1e-3)
        for k in range(n):
            samples_tb[k].append(times[k])
    layers = tuple(LayerProfile(k + 1, params[k].numel(), statistics.median(samples_tb[k][1:])) for k in range(n))
    widths = {p.element_size() for p in params}
    return ModelProfile(name=name, layers=layers, forward_time=statistics.median(samples_tf[1:]),
                        element_bytes=widths.pop() if len(widths) == 1 else 4)
