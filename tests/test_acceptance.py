"""The reference's numbered acceptance criteria (/root/reference/pkg/tests/test_acceptance.py),
run against this implementation.  Criteria 7 and 8 exercise the data path and live
in test_gpu_multi.py."""

import math
import random
import time

from conftest import ACCEPTANCE_SEED, draw_instance, draw_mixed_instance, golden_planner, greedy_gap_instance, make_profile
from paper_1811_11141_b200 import (
    Collective,
    CollectiveParams,
    CommModel,
    Measurement,
    MergePlan,
    OverlapCase,
    Strategy,
    allreduce_time,
    brute_force_plan,
    classify_case,
    derive_ab,
    find_merge_plan,
    fit_ab,
    resnet50_like,
    simulate_mgwfbp,
    simulate_naive,
    simulate_sync_easgd,
    simulate_wfbp,
    sweep,
)


def test_criterion_1_startup_calibration():
    for n, want in {2: 90.52e-6, 4: 271.56e-6, 8: 633.64e-6}.items():
        got = derive_ab(CollectiveParams(Collective.RING, n, 45.26e-6, 0.0, 0.0)).a
        assert abs(got - want) <= math.ulp(want)


def test_criterion_2_superadditive_gap():
    rng = random.Random(ACCEPTANCE_SEED)
    for _ in range(10_000):
        a = rng.randrange(1, 1 << 24) / (1 << 20)
        b = rng.randrange(0, 1 << 24) / (1 << 44)
        m1, m2 = 1 << rng.randrange(0, 26), 1 << rng.randrange(0, 26)
        model = CommModel(a=a, b=b)
        assert allreduce_time(m1, model) + allreduce_time(m2, model) - allreduce_time(m1 + m2, model) == a


def test_criterion_3_same_counterexamples_as_reference():
    """Greedy vs exhaustive on the reference's frozen 1000-instance stream: the
    disagreements are exactly the 102 the reference archived (index for index,
    bit-identical t_iter), and all three overlap regimes occur."""
    archived = {c["index"]: c for c in golden_planner()["archive"]["cases"]}
    rng = random.Random(ACCEPTANCE_SEED)
    found, cases = {}, set()
    for index in range(1000):
        profile, model = draw_instance(rng)
        cases.add(classify_case(profile, model))
        greedy = find_merge_plan(profile, model)
        oracle = brute_force_plan(profile, model)
        tg = simulate_mgwfbp(profile, model, greedy).t_iter
        to = simulate_mgwfbp(profile, model, oracle).t_iter
        if tg != to:
            found[index] = (sorted(greedy.merged_layers), sorted(oracle.merged_layers), tg, to)
    assert cases >= {OverlapCase.CASE_1, OverlapCase.CASE_2, OverlapCase.CASE_3}
    assert set(found) == set(archived)
    for index, (gp, op, tg, to) in found.items():
        c = archived[index]
        assert (gp, op, tg, to) == (c["greedy_plan"], c["oracle_plan"], c["greedy_t_iter"], c["oracle_t_iter"])


def _adversarial():
    out = []
    for a in (1e-9, 1e-7, 1e-5, 1e-3, 1e-1, 1e1, 1e3):
        out.append((make_profile([1000] * 6, [1e-3] * 6, 1e-3), CommModel(a=a, b=1e-9)))
    for b in (0.0, 1e-13, 1e-11, 1e-9):
        out.append((make_profile([10 ** k for k in range(1, 7)], [1e-3] * 6, 2e-3), CommModel(a=1e-4, b=b)))
    for scale in (0.25, 0.5, 0.999, 1.0, 1.001, 2.0, 8.0):
        out.append((make_profile([100, 100], [scale * 1e-3, 1e-3], 1e-3), CommModel(a=1e-3, b=1e-9)))
    for L in (2, 3, 6, 12):
        out.append((make_profile([500] * L, [1e-3] * L, 0.0), CommModel(a=5e-4, b=1e-9)))
    for pos in range(5):
        params = [100] * 5
        params[pos] = 5_000_000
        out.append((make_profile(params, [2e-3] * 5, 1e-3), CommModel(a=1e-3, b=2e-9)))
    for L in (2, 4, 8, 12):
        out.append((make_profile([1024] * L, [2.0 ** -10] * L, 2.0 ** -8), CommModel(a=2.0 ** -10, b=2.0 ** -22)))
    wp, wm = greedy_gap_instance()
    out.append((wp, wm))
    for k in range(1, 8):
        out.append((wp, CommModel(a=wm.a * 2.0 ** (k - 3), b=wm.b * 2.0 ** (3 - k))))
    for L in (4, 8, 16):
        asc = [10 ** (1 + i % 6) for i in range(L)]
        down = [1e-2 / (i + 1) for i in range(L)]
        out.append((make_profile(asc, down, 1e-2), CommModel(a=1e-4, b=1e-9)))
        out.append((make_profile(asc[::-1], down[::-1], 1e-2), CommModel(a=1e-4, b=1e-9)))
    for L in (2, 4, 8, 12, 16):
        out.append((make_profile([3_000_000] * L, [1e-5] * L, 1e-5), CommModel(a=1e-3, b=4e-9)))
        out.append((make_profile([10] * L, [5e-2] * L, 5e-2), CommModel(a=1e-6, b=1e-10)))
    return out


def test_criterion_4_strategy_dominance():
    rng = random.Random(ACCEPTANCE_SEED)
    instances = [draw_instance(rng) for _ in range(1000)] + _adversarial()
    for profile, model in instances:
        mg = simulate_mgwfbp(profile, model, find_merge_plan(profile, model)).t_iter
        wfbp = simulate_wfbp(profile, model).t_iter
        assert mg <= wfbp and mg <= simulate_sync_easgd(profile, model).t_iter
        assert wfbp <= simulate_naive(profile, model).t_iter


def test_criterion_5_degeneracy_identities():
    rng = random.Random(ACCEPTANCE_SEED + 5)
    for i in range(200):
        profile, model = draw_mixed_instance(rng) if i % 2 else draw_instance(rng)
        n = profile.num_layers
        w, e = simulate_wfbp(profile, model), simulate_mgwfbp(profile, model, MergePlan(frozenset(), n))
        s, f = simulate_sync_easgd(profile, model), simulate_mgwfbp(profile, model, MergePlan(frozenset(range(2, n + 1)), n))
        assert (w.tau_c, w.t_c, w.comm_end, w.t_iter, w.t_c_no) == (e.tau_c, e.t_c, e.comm_end, e.t_iter, e.t_c_no)
        assert (s.tau_c, s.t_c, s.comm_end, s.t_iter, s.t_c_no) == (f.tau_c, f.t_c, f.comm_end, f.t_iter, f.t_c_no)


def test_criterion_6_scaling_shape():
    params = CollectiveParams(Collective.RING, 4, 45.26e-6, 8e-10, 5e-11)
    n_list = [4, 8, 16, 32, 64]
    result = sweep(resnet50_like(), params, n_list)
    w = {n: result.t_iter(n, Strategy.WFBP) for n in n_list}
    s = {n: result.t_iter(n, Strategy.SYNC_EASGD) for n in n_list}
    m = {n: result.t_iter(n, Strategy.MGWFBP) for n in n_list}
    assert w[4] < s[4] and w[8] < s[8] and s[64] < w[64]
    assert all(m[n] <= min(w[n], s[n]) for n in n_list)
    assert 1.3 <= w[64] / m[64] <= 2.2


def test_criterion_9_fit_recovery():
    truth = CommModel(a=3e-4, b=2e-9)
    sizes = [1 << k for k in range(12, 24)]
    f0 = fit_ab([Measurement(m, allreduce_time(m, truth), 4) for m in sizes])
    assert max(abs(f0.a - truth.a) / truth.a, abs(f0.b - truth.b) / truth.b) < 1e-10
    rng = random.Random(0)
    noisy = [Measurement(m, allreduce_time(m, truth) * (1 + rng.uniform(-0.02, 0.02)), 4) for m in sizes for _ in range(5)]
    f1 = fit_ab(noisy)
    assert max(abs(f1.a - truth.a) / truth.a, abs(f1.b - truth.b) / truth.b) < 0.05
