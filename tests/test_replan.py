"""Online re-planning: live (a, b) refits drive Algorithm 1 again.
CPU only; the multi-rank agreement runs under gloo with world_size 2."""

import multiprocessing as mp
import os

import pytest

from paper_1811_11141_b200 import CommModel, find_merge_plan, resnet50_like
from paper_1811_11141_b200.allreduce_net import _free_port
from paper_1811_11141_b200.replan import OnlinePlanner

PROFILE = resnet50_like(backward_seconds=0.00972, forward_seconds=0.00464)  # B200-class timings
SIZES = [1 << k for k in range(12, 27)]


def feed(planner, model, reps=2):
    for _ in range(reps):
        for m in SIZES:
            planner.observe(m, model.allreduce_time(m))


def test_first_fit_plans_like_the_offline_workflow():
    live = CommModel(12e-6, 1 / 500e9)
    p = OnlinePlanner(PROFILE, 4, min_samples=8)
    assert p.update() is None  # nothing observed yet
    feed(p, live)
    plan = p.update()
    assert p.model is not None and abs(p.model.a - live.a) < 1e-9 and abs(p.model.b - live.b) < 1e-15
    assert (plan or p.plan) == find_merge_plan(PROFILE, p.model)


def test_drift_past_threshold_replans_and_small_noise_does_not():
    fast = CommModel(12e-6, 1 / 500e9)
    p = OnlinePlanner(PROFILE, 4, model=fast, window=len(SIZES) * 2, min_samples=8, threshold=0.1)
    first = p.plan
    feed(p, CommModel(12.5e-6, 1 / 490e9))  # within 10 %: keep the plan
    assert p.update() is None and p.plan == first and p.model == fast
    slow = CommModel(400e-6, 1 / 50e9)  # a congested fabric: startup dominates
    feed(p, slow)
    plan = p.update()
    assert plan is not None and p.replans == 1
    assert plan == find_merge_plan(PROFILE, p.model)
    assert len(plan.groups()) < len(first.groups())  # a larger `a` merges more


def test_negative_slope_window_keeps_the_plan():
    p = OnlinePlanner(PROFILE, 2, min_samples=4)
    for m, s in ((4096, 4e-5), (8192, 3e-5), (16384, 2e-5), (32768, 1e-5)):
        p.observe(m, s)
    assert p.update() is None and p.model is None


def test_validation():
    with pytest.raises(ValueError):
        OnlinePlanner(PROFILE, 1)
    with pytest.raises(ValueError):
        OnlinePlanner(PROFILE, 2, threshold=0)
    with pytest.raises(ValueError):
        OnlinePlanner(PROFILE, 2, window=4, min_samples=8)
    p = OnlinePlanner(PROFILE, 2)
    p.observe(0, 1e-5)  # silent group: nothing was sent
    p.observe(4096, 0.0)
    assert len(p.samples) == 0


def _agree_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1811_11141_b200.replan import dist_agree

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = OnlinePlanner(PROFILE, world, min_samples=8, agree=dist_agree())
        # rank 1 sees a slower fabric than rank 0: both must adopt the max (a, b)
        feed(p, CommModel(20e-6 if rank == 0 else 300e-6, 1 / (500e9 if rank == 0 else 100e9)))
        plan = p.update()
        q.put((rank, (p.model.a, p.model.b), sorted((plan or p.plan).merged_layers)))
    finally:
        dist.destroy_process_group()


def test_ranks_agree_on_one_plan_over_gloo():
    world = 2
    port = _free_port("127.0.0.1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict((r, (m, plan)) for r, m, plan in (q.get(timeout=120) for _ in range(world)))
    for pr in procs:
        pr.join(timeout=10)
    assert res[0] == res[1]
    (a, b), merged = res[0]
    assert a == pytest.approx(300e-6, rel=1e-6) and b == pytest.approx(1 / 100e9, rel=1e-6)
    assert merged == sorted(find_merge_plan(PROFILE, CommModel(a, b)).merged_layers)


def test_calibrate_startup_picks_the_fastest_measured_scale():
    from paper_1811_11141_b200.replan import calibrate_startup

    model = CommModel(12e-6, 1 / 500e9)
    calls = []

    def measure(plan):  # a synthetic "real step": every collective costs 20 µs of interference
        calls.append(plan.merged_layers)
        groups = len(plan.groups())
        return 15e-3 + groups * 20e-6 + (300e-6 if groups == 1 else 0.0)

    k, plan, times = calibrate_startup(PROFILE, model, measure, scales=(1, 4, 16, 64, 256))
    assert len(calls) == len(set(calls))  # identical plans are measured once
    assert times[k] == min(times.values())
    assert plan == find_merge_plan(PROFILE, CommModel(model.a * k, model.b))
    assert len(plan.groups()) < len(find_merge_plan(PROFILE, model).groups())
