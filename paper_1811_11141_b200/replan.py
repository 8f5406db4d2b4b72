"""Online re-planning from live (a, b) fits.

The reference plans once: calibrate (``bench_allreduce`` -> ``fit_ab``,
``comm_model.py:182-218``), then ``find_merge_plan`` (``merge_planner.py:150-180``),
then run.  On a shared NVSwitch the startup ``a`` and per-byte ``b`` drift with
load (other jobs, the overlapped backward's SM/HBM pressure), so ``OnlinePlanner``
keeps a sliding window of the group exchanges the iteration actually performed --
(bucket bytes, device seconds from the kernels' own ``%globaltimer`` stamps) -- refits
(a, b) with the reference's OLS, and re-runs Algorithm 1 when the fitted model moved
by more than ``threshold``.  Every rank must switch plans at the same iteration with
the same plan (the collectives of a plan are matched across ranks), so the fitted
model goes through ``agree`` first: ``dist_agree`` takes the element-wise maximum of
(a, b) over ranks (the slowest rank sets the pace of every collective).

The plan is a pure function of (profile, model), so equal models give equal plans on
every rank without shipping the plan itself.
"""

from __future__ import annotations

import collections
from typing import Callable, Iterable

from .comm_model import CommModel, Measurement, fit_ab
from .merge_planner import MergePlan, find_merge_plan
from .model_profile import ModelProfile

__all__ = ["OnlinePlanner", "calibrate_startup", "dist_agree", "dist_max", "observe_iteration"]


def dist_agree(group=None) -> Callable[[CommModel], CommModel]:
    """(a, b) max-reduced over the ranks of a torch.distributed group (any backend)."""

    def agree(model: CommModel) -> CommModel:
        import torch
        import torch.distributed as dist

        backend = dist.get_backend(group)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        t = torch.tensor([model.a, model.b], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return CommModel(float(t[0]), float(t[1]))

    return agree


def dist_max(group=None) -> Callable[[float], float]:
    """A float max-reduced over the ranks of a torch.distributed group."""

    def agree(x: float) -> float:
        import torch
        import torch.distributed as dist

        backend = dist.get_backend(group)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t[0])

    return agree


def calibrate_startup(profile: ModelProfile, model: CommModel, measure: Callable[[MergePlan], float], *,
                      scales=(1, 2, 4, 8, 16, 32, 64), agree: Callable[[float], float] | None = None):
    """Interference-aware startup for real overlap.

    The alpha/beta model prices an exchange alone; overlapped with a real backward pass
    every collective also takes SMs and HBM from the backward kernels, a per-collective
    cost the model does not see.  Pricing it as a larger startup ``k * a`` lets Algorithm 1
    trade it off (fewer, larger messages).  ``measure(plan)`` returns the seconds of a real
    training step under ``plan`` (collective across ranks when ``agree`` is set: it is
    called with the same plans in the same order on every rank); plans that coincide are
    measured once.  Returns ``(k, plan, {k: seconds})`` for the fastest ``k``.
    """
    times: dict[float, float] = {}
    by_plan: dict[frozenset, float] = {}
    for k in scales:
        plan = find_merge_plan(profile, CommModel(model.a * k, model.b))
        key = plan.merged_layers
        if key not in by_plan:
            t = float(measure(plan))
            by_plan[key] = agree(t) if agree is not None else t
        times[k] = by_plan[key]
    best = min(scales, key=lambda k: (times[k], k))
    return best, find_merge_plan(profile, CommModel(model.a * best, model.b)), times


class OnlinePlanner:
    """Sliding-window (a, b) fit over live group exchanges, re-planning on drift.

    ``observe(nbytes, seconds)`` per exchanged group (zero-byte groups are ignored:
    nothing is sent for them, ``allreduce_net.py:549``); ``update()`` once per iteration
    at the same point on every rank returns the new plan when it changed, else None.
    """

    def __init__(self, profile: ModelProfile, n_nodes: int, *, model: CommModel | None = None,
                 plan: MergePlan | None = None, window: int = 512, min_samples: int = 16,
                 threshold: float = 0.10, agree: Callable[[CommModel], CommModel] | None = None):
        if n_nodes < 2:
            raise ValueError("online re-planning needs >= 2 nodes (there is no exchange at N=1)")
        if not 0 < threshold:
            raise ValueError(f"threshold must be > 0, got {threshold!r}")
        if min_samples < 2 or window < min_samples:
            raise ValueError("need window >= min_samples >= 2")
        self.profile = profile
        self.n_nodes = n_nodes
        self.samples: collections.deque[Measurement] = collections.deque(maxlen=window)
        self.min_samples = min_samples
        self.threshold = threshold
        self.agree = agree
        self.model = model
        self.plan = plan if plan is not None else (find_merge_plan(profile, model) if model is not None else None)
        self.replans = 0

    def observe(self, nbytes: int, seconds: float) -> None:
        if nbytes > 0 and seconds > 0:
            self.samples.append(Measurement(int(nbytes), float(seconds), self.n_nodes))

    def observe_many(self, pairs: Iterable[tuple[int, float]]) -> None:
        for nbytes, seconds in pairs:
            self.observe(nbytes, seconds)

    def _fit(self) -> CommModel | None:
        if len(self.samples) < self.min_samples or len({s.nbytes for s in self.samples}) < 2:
            return None
        try:
            return fit_ab(list(self.samples))
        except ValueError:  # negative slope: the window contradicts the model; keep the plan
            return None

    def _moved(self, new: CommModel) -> bool:
        old = self.model
        if old is None:
            return True

        def rel(x, y):
            return abs(x - y) / max(abs(y), 1e-30)

        return rel(new.a, old.a) > self.threshold or rel(new.b, old.b) > self.threshold

    def update(self) -> MergePlan | None:
        """Refit; if (a, b) moved past the threshold, re-plan.  Collective when ``agree``
        is set: every rank must call it at the same iteration."""
        fitted = self._fit()
        if self.agree is not None:
            # ranks that cannot fit yet still take part in the reduction (with a sentinel
            # of their current model) so the collective never deadlocks
            fitted = self.agree(fitted if fitted is not None else (self.model or CommModel(0.0, 0.0)))
            if fitted.a == 0.0 and fitted.b == 0.0:
                return None
        if fitted is None or not self._moved(fitted):
            return None
        self.model = fitted
        plan = find_merge_plan(self.profile, fitted)
        if plan == self.plan:
            return None
        self.plan = plan
        self.replans += 1
        return plan


def observe_iteration(planner: OnlinePlanner, iteration) -> None:
    """Feed one ``OverlappedIteration``'s per-group exchange spans into ``planner``
    (the fused kernel's span, or pack + all-reduce + unpack when unfused)."""
    pack, ar, unpack = iteration.kernel_times()
    for nbytes, p, a, u in zip(iteration.group_bytes(), pack, ar, unpack):
        planner.observe(nbytes, p + a + u)
