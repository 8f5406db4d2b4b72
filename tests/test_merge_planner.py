"""Merge-schedule solver: bit-exact with the reference on its archived counterexamples
and on reference-generated fixtures; behaviour pins from the reference suite
(/root/reference/pkg/tests/test_merge_planner.py)."""

import io
import random

import pytest

from conftest import (
    draw_instance,
    draw_mixed_instance,
    golden_planner,
    greedy_gap_instance,
    make_profile,
    worked_instance,
)
from paper_1811_11141_b200 import (
    CommModel,
    MergePlan,
    PlannerState,
    apply_merge,
    backward_start_times,
    brute_force_plan,
    calculate_comm_start,
    comm_start_times,
    find_merge_plan,
    load_plan,
    resnet50_like,
    googlenet_like,
    save_plan,
    simulate_mgwfbp,
    simulate_sync_easgd,
    simulate_wfbp,
    synth_profile,
)
from paper_1811_11141_b200.merge_planner import _iteration_time


def _profile(case):
    return make_profile(case["params"], case["backward_times"], case["forward_time"], case.get("element_bytes", 4))


def test_archived_counterexamples_bit_exact():
    """The 102 instances the reference archived (criterion 3): same greedy plan,
    same brute-force plan, same t_iter doubles."""
    cases = golden_planner()["archive"]["cases"]
    assert len(cases) == 102
    for c in cases:
        profile, model = _profile(c), CommModel(c["a"], c["b"])
        greedy = find_merge_plan(profile, model)
        assert sorted(greedy.merged_layers) == c["greedy_plan"]
        assert simulate_mgwfbp(profile, model, greedy).t_iter == c["greedy_t_iter"]
        brute = brute_force_plan(profile, model)
        assert sorted(brute.merged_layers) == c["oracle_plan"]
        assert simulate_mgwfbp(profile, model, brute).t_iter == c["oracle_t_iter"]
        assert simulate_wfbp(profile, model).t_iter == c["wfbp_t_iter"]
        assert simulate_sync_easgd(profile, model).t_iter == c["synceasgd_t_iter"]


def test_reference_generated_plans_bit_exact():
    for c in golden_planner()["random"]:
        profile, model = _profile(c), CommModel(c["a"], c["b"])
        plan = find_merge_plan(profile, model)
        assert sorted(plan.merged_layers) == c["plan"]
        assert [list(g) for g in plan.groups()] == c["groups"]
        if "brute_plan" in c:
            assert sorted(brute_force_plan(profile, model).merged_layers) == c["brute_plan"]


@pytest.mark.parametrize("key", ["resnet50_like", "resnet50_like_fast", "googlenet_like", "synth_1000", "synth_12x5"])
def test_named_profile_plans_bit_exact(key):
    g = golden_planner()["named"][key]
    profile = make_profile(g["params"], g["backward_times"], g["forward_time"], name=g["name"])
    for row in g["plans"]:
        model = CommModel(row["a"], row["b"])
        plan = find_merge_plan(profile, model)
        assert sorted(plan.merged_layers) == row["plan"]
        assert simulate_mgwfbp(profile, model, plan).t_iter == row["mgwfbp_t_iter"]
        assert simulate_wfbp(profile, model).t_iter == row["wfbp_t_iter"]
        assert simulate_sync_easgd(profile, model).t_iter == row["synceasgd_t_iter"]


def _replay_full_recompute(profile, model):
    """The reference's loop shape (merge_planner.py:164-180): full tau_c recompute
    after every accepted merge.  Used to pin the O(L) lazy sweep against it."""
    n = profile.num_layers
    if model.a == 0.0:
        return frozenset()
    t_b = profile.backward_times()
    tau_b = backward_start_times(profile)
    virtual = tau_b[0] + t_b[0]
    state = PlannerState.from_profile(profile, model)
    tau_c = comm_start_times(state.t_c, t_b, tau_b)
    merged = set()
    for layer in range(n, 1, -1):
        if state.params[layer - 1] == 0 or state.params[layer - 2] == 0:
            continue
        below = tau_b[layer - 3] if layer >= 3 else virtual
        if below - tau_c[layer - 1] < model.a:
            apply_merge(state, layer)
            merged.add(layer)
            tau_c = comm_start_times(state.t_c, t_b, tau_b)
    return frozenset(merged)


def test_lazy_sweep_equals_full_recompute():
    rng = random.Random(2024)
    for k in range(400):
        maker = draw_mixed_instance if k % 2 else draw_instance
        profile, model = maker(rng, (12, 40, 150)[k % 3])
        assert find_merge_plan(profile, model).merged_layers == _replay_full_recompute(profile, model)
    big = synth_profile(1000, param_range=(1024, 16_777_216), seed=0)
    for a, b in ((2e-5, 1.6e-12), (4e-4, 1e-11), (1e-2, 1e-9)):
        model = CommModel(a, b)
        assert find_merge_plan(big, model).merged_layers == _replay_full_recompute(big, model)


def test_merge_plan_validation_and_groups():
    MergePlan(frozenset(), 1)
    for bad in ({1}, {4}):
        with pytest.raises(ValueError):
            MergePlan(frozenset(bad), 3)
    with pytest.raises(ValueError):
        MergePlan(frozenset(), 0)
    plan = MergePlan(frozenset({2, 5}), 6)
    assert plan.groups() == [(1, 2), (3, 3), (4, 5), (6, 6)]
    assert (plan.head_of(2), plan.head_of(5), plan.head_of(6)) == (1, 4, 6)
    assert MergePlan(frozenset(range(2, 7)), 6).groups() == [(1, 6)]
    assert MergePlan(frozenset(), 4).groups() == [(1, 1), (2, 2), (3, 3), (4, 4)]
    with pytest.raises(ValueError):
        plan.head_of(7)


def test_plan_round_trip(tmp_path):
    plan = MergePlan(frozenset({2, 4, 7}), 8)
    path = tmp_path / "plan.json"
    save_plan(plan, path)
    assert load_plan(path, 8) == plan
    assert path.read_text() == "[2, 4, 7]\n"
    buf = io.StringIO()
    save_plan(plan, buf)
    buf.seek(0)
    assert load_plan(buf, 8) == plan
    (tmp_path / "bad.json").write_text('{"merged": [2]}')
    with pytest.raises(ValueError):
        load_plan(tmp_path / "bad.json", 8)


def test_apply_merge_folds_mass_down():
    state = PlannerState.from_profile(make_profile([10, 20, 30], [1e-3] * 3, 1e-3), CommModel(a=1e-3, b=1e-9))
    apply_merge(state, 3)
    assert state.params == [10, 50, 0] and state.t_c[2] == 0.0
    assert state.t_c[1] == 1e-3 + 1e-9 * (4 * 50)
    for bad in (1, 4):
        with pytest.raises(ValueError):
            apply_merge(state, bad)


def test_worked_instance_plan_is_layer_two():
    profile, model = worked_instance()
    plan = find_merge_plan(profile, model)
    assert plan.merged_layers == frozenset({2})
    assert simulate_mgwfbp(profile, model, plan).t_iter == 15.5
    assert brute_force_plan(profile, model) == plan


def test_zero_startup_and_huge_startup():
    rng = random.Random(3)
    for _ in range(50):
        profile, model = draw_instance(rng)
        assert find_merge_plan(profile, CommModel(a=0.0, b=model.b)).merged_layers == frozenset()
    profile = make_profile([100, 200, 300, 400], [1e-3] * 4, 1e-3)
    model = CommModel(a=10.0, b=1e-9)
    plan = find_merge_plan(profile, model)
    assert plan.merged_layers == frozenset({2, 3, 4})
    assert simulate_mgwfbp(profile, model, plan).t_iter == simulate_sync_easgd(profile, model).t_iter


def test_silent_layer_rules():
    rng = random.Random(17)
    for _ in range(300):
        profile, model = draw_mixed_instance(rng)
        plan = find_merge_plan(profile, model)
        counts = profile.param_counts()
        for layer in plan.merged_layers:
            assert counts[layer - 1] > 0 and counts[plan.head_of(layer) - 1] > 0
    profile = make_profile([1000, 0, 1000], [1e-4] * 3, 1e-3)
    model = CommModel(a=0.01, b=1e-9)
    assert find_merge_plan(profile, model).merged_layers == frozenset()
    squeezed = make_profile([1000, 1000], [1e-4, 1e-4], 1e-3)
    assert find_merge_plan(squeezed, model).merged_layers == frozenset({2})


def test_dominance_over_both_baselines():
    rng = random.Random(31)
    for _ in range(400):
        profile, model = draw_instance(rng)
        mg = simulate_mgwfbp(profile, model, find_merge_plan(profile, model)).t_iter
        assert mg <= simulate_wfbp(profile, model).t_iter
        assert mg <= simulate_sync_easgd(profile, model).t_iter


def test_greedy_gap_witness():
    profile, model = greedy_gap_instance()
    greedy, brute = find_merge_plan(profile, model), brute_force_plan(profile, model)
    assert greedy.merged_layers == frozenset({3, 4, 5})
    assert brute.merged_layers == frozenset({2, 3, 4})
    tg = simulate_mgwfbp(profile, model, greedy).t_iter
    tb = simulate_mgwfbp(profile, model, brute).t_iter
    assert tb < tg and (tg - tb) / tb > 0.02


def test_brute_force_tie_breaking_and_guards():
    assert brute_force_plan(make_profile([1], [1e-3], 1e-3), CommModel(a=1.0, b=0.0)).merged_layers == frozenset()
    silent = make_profile([1000, 0, 0], [1e-3] * 3, 1e-3)
    assert brute_force_plan(silent, CommModel(a=1.0, b=1e-9)).merged_layers == frozenset()
    big = make_profile([1] * 17, [1e-3] * 17, 1e-3)
    with pytest.raises(ValueError):
        brute_force_plan(big, CommModel(a=1e-3, b=1e-9))


def test_collapsed_evaluator_matches_full_timeline():
    rng = random.Random(43)
    for _ in range(60):
        profile, model = draw_mixed_instance(rng, max_layers=7)
        n = profile.num_layers
        t_b = profile.backward_times()
        ready = [tb + s for tb, s in zip(t_b, backward_start_times(profile))]
        for mask in range(1 << (n - 1)):
            fast = _iteration_time(ready, profile.param_counts(), 4, model.a, model.b, mask)
            plan = MergePlan(frozenset(k + 2 for k in range(n - 1) if (mask >> k) & 1), n)
            assert fast == simulate_mgwfbp(profile, model, plan).t_iter


def test_comm_start_alias():
    assert calculate_comm_start is comm_start_times


def test_planner_is_linear_time():
    """O(L) sweep: a 1000-layer profile with many merges plans in milliseconds."""
    import time

    big = synth_profile(1000, param_range=(1024, 16_777_216), seed=0)
    model = CommModel(a=5e-3, b=1e-12)  # merges almost everything
    t0 = time.perf_counter()
    plan = find_merge_plan(big, model)
    elapsed = time.perf_counter() - t0
    assert len(plan.merged_layers) > 500
    assert elapsed < 0.05
