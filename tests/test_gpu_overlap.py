"""Algorithm 2 on streams (single GPU): the iteration engine reproduces the simulated
compute timeline, verifies the reference's expected values, and the graph replay
matches eager execution."""

import pytest

from paper_1811_11141_b200 import CommModel, MergePlan, find_merge_plan, resnet50_like, simulate_mgwfbp, synth_profile  # noqa: F401
from paper_1811_11141_b200.overlap import OverlappedIteration

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    return torch


def _plans(profile):
    n = profile.num_layers
    model = CommModel(a=2e-5, b=1.5e-12)
    return {
        "wfbp": MergePlan(frozenset(), n),
        "synceasgd": MergePlan(frozenset(range(2, n + 1)), n),
        "mgwfbp": find_merge_plan(profile, model),
    }


@pytest.mark.parametrize("graph", [False, True])
def test_single_gpu_iteration_matches_profile(torch_cuda, graph):
    profile = resnet50_like(backward_seconds=4e-3, forward_seconds=2e-3)
    compute = profile.forward_time + profile.total_backward_time
    for name, plan in _plans(profile).items():
        it = OverlappedIteration(profile, plan, comm=None, rank=0, world=1, device="cuda:0", graph=graph, fused=graph)
        try:
            for _ in range(3):
                t = it.run()
            assert it.verify(), name
            assert abs(t.compute_time - compute) / compute < 0.02, (name, t)
            assert t.t_iter >= t.compute_time
            assert 0.0 <= t.t_c_no < 2e-3, (name, t)
            assert len(t.group_comm) == len(plan.groups())
        finally:
            it.close()


def test_host_io_end_to_end(torch_cuda):
    profile = resnet50_like(backward_seconds=8e-3, forward_seconds=4e-3)
    it = OverlappedIteration(profile, MergePlan(frozenset(), profile.num_layers), comm=None, rank=0, world=1,
                             device="cuda:0", fill=False, host_io=True)
    try:
        it.run()
        assert it.verify()
        assert it.io_bytes() == (4 * profile.total_params, 4 * profile.total_params)
    finally:
        it.close()


def test_many_small_groups_graph(torch_cuda):
    profile = synth_profile(300, param_range=(1024, 65536), time_scale=2e-5, seed=3)
    it = OverlappedIteration(profile, None, comm=None, rank=0, world=1, device="cuda:0", graph=True)
    try:
        for _ in range(3):
            t = it.run()
        assert it.verify()
        assert t.t_iter >= t.compute_time
    finally:
        it.close()


def test_launch_count_reported(torch_cuda):
    profile = resnet50_like(backward_seconds=4e-3, forward_seconds=2e-3)
    it = OverlappedIteration(profile, None, comm=None, rank=0, world=1, device="cuda:0")
    try:
        # stamp reset + mark + per group: spin, fill, pack, unpack
        assert it.launches_per_iteration == 2 + 4 * profile.num_layers
    finally:
        it.close()
    it = OverlappedIteration(profile, None, comm=None, rank=0, world=1, device="cuda:0", fused=True)
    try:
        # per group: spin, fill, one fused kernel
        assert it.launches_per_iteration == 2 + 3 * profile.num_layers
        it.run()
        assert it.verify()
    finally:
        it.close()


def test_autograd_sync_single_gpu(torch_cuda):
    """Hooks fire for every parameter, groups complete, and the scale is applied once."""
    torch = torch_cuda
    from paper_1811_11141_b200.autograd import MergedGradientSync, measure_profile, trainable_parameters

    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.ReLU(), torch.nn.Linear(128, 10)).cuda()
    x = torch.randn(32, 64, device="cuda")
    step = lambda: net(x).square().mean()  # noqa: E731
    params = trainable_parameters(net)
    prof = measure_profile(net, step, repeats=2)
    assert prof.num_layers == 4 and prof.total_params == sum(p.numel() for p in params)
    net.zero_grad(set_to_none=False)
    step().backward()
    want = [p.grad.clone() * 0.5 for p in params]
    sync = MergedGradientSync(params, MergePlan(frozenset({2, 4}), 4), scale=0.5)
    try:
        net.zero_grad(set_to_none=False)
        step().backward()
        sync.finish()
        assert sync.launched == 2
        for p, w in zip(params, want):
            assert torch.equal(p.grad, w)
    finally:
        sync.close()


@pytest.mark.parametrize("graph", [False, True])
def test_bf16_engine_single_gpu(torch_cuda, graph):
    """Algorithm 2 on bf16 gradients (MGW_SCHED_BF16: bf16 fill, the bf16 group kernel with
    fp32 accumulation): every plan verifies the reference's exact sums, timeline as fp32."""
    torch = torch_cuda
    profile = resnet50_like(backward_seconds=4e-3, forward_seconds=2e-3)
    compute = profile.forward_time + profile.total_backward_time
    for name, plan in _plans(profile).items():
        it = OverlappedIteration(profile, plan, comm=None, rank=0, world=1, device="cuda:0", graph=graph, fused=True,
                                 dtype=torch.bfloat16)
        try:
            for _ in range(3):
                t = it.run()
            assert it.verify(), name
            assert abs(t.compute_time - compute) / compute < 0.02, (name, t)
            assert it.group_bytes()[0] == 2 * sum(p for _, p, _ in it.layout[0][2])
        finally:
            it.close()
    with pytest.raises(ValueError):
        OverlappedIteration(profile, None, comm=None, rank=0, world=1, device="cuda:0", host_io=True,
                            dtype=torch.bfloat16)


@pytest.mark.parametrize("plan_name", ["wfbp", "mgwfbp", "synceasgd"])
def test_measured_timeline_events(torch_cuda, plan_name):
    """The engine's own stamps give a measured Timeline (schedule_sim.py:65-100): one
    backward row per layer, one comm row per sending group (at its head layer), every
    exchange starting after its gradients were produced, t_iter >= compute, and the
    measured compute / exposed time close to the event-timed IterationTimes."""
    from paper_1811_11141_b200.schedule_sim import Timeline

    profile = resnet50_like(backward_seconds=4e-3, forward_seconds=2e-3)
    plan = _plans(profile)[plan_name]
    it = OverlappedIteration(profile, plan, comm=None, rank=0, world=1, device="cuda:0", graph=True, fused=True)
    try:
        for _ in range(3):
            times = it.run()
        tl = it.measured_timeline()
    finally:
        it.close()
    assert isinstance(tl, Timeline)
    rows = tl.events(profile)
    back = [r for r in rows if r[1] == "backward"]
    comm = [r for r in rows if r[1] == "comm"]
    assert len(back) == profile.num_layers
    assert {r[0] for r in comm} == {low for low, _ in plan.groups()}
    for layer, _, t0, t1 in comm:
        ready = tl.tau_b[layer - 1] + profile.backward_times()[layer - 1]
        assert t0 >= ready - 1e-6 and t1 >= t0, (layer, t0, ready)
    assert tl.t_iter >= tl.compute_time
    assert abs(tl.compute_time - times.compute_time) < 5e-5
    assert abs(tl.t_c_no - times.t_c_no) < 2e-5
