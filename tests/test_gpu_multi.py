"""The reference's collective and emulation tests, run through the real multi-process
CUDA-IPC path (one process per GPU).  Skipped unless >= 2 GPUs are visible; run with
`gpurun --gpus 2|4 -- python -m pytest tests -m gpu`."""

from functools import partial

import numpy as np
import pytest

import _mp_tasks
from conftest import ROOT, cuda_devices, golden_ring, make_profile
from paper_1811_11141_b200 import (
    CommModel,
    EmulationReport,
    MergePlan,
    bench_local,
    emulate_local,
    find_merge_plan,
    fit_ab,
    resnet50_like,
    run_workers,
    simulate_mgwfbp,
    synth_profile,
)

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.fixture(autouse=True)
def _two_gpus():
    if cuda_devices() < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU)")


def _worlds():
    n = cuda_devices()
    return [w for w in (2, 3, 4, 8) if w <= n]


def test_exact_sums_and_counters():
    for n in _worlds():
        results = run_workers(n, _mp_tasks.sum_task)
        assert set(results) == set(range(n))
        assert all(frames == 2 for frames in results.values())


def test_payload_smaller_than_group():
    n = max(_worlds())
    assert all(run_workers(n, _mp_tasks.single_element_task).values())


def test_empty_and_fewer_elements_than_ranks():
    for n in _worlds():
        for verdicts in run_workers(n, _mp_tasks.empty_and_tiny_task).values():
            assert all(verdicts), verdicts


def test_length_mismatch_is_a_protocol_error():
    with pytest.raises(RuntimeError) as err:
        run_workers(2, _mp_tasks.mismatched_task, timeout=60)
    assert "buffer lengths" in str(err.value) or "ProtocolError" in str(err.value)


def test_dtype_mismatch_is_a_protocol_error():
    """bf16 on one rank, fp32 on another (same length): caught by the barrier / LL header tag."""
    with pytest.raises(RuntimeError) as err:
        run_workers(2, _mp_tasks.dtype_mismatch_task, timeout=60)
    assert "buffer lengths" in str(err.value) or "ProtocolError" in str(err.value)


def test_absent_peer_times_out_as_protocol_error():
    """A peer that never reaches the collective: bounded spin -> ProtocolError, not a hang."""
    import time

    t0 = time.monotonic()
    with pytest.raises(RuntimeError) as err:
        run_workers(2, _mp_tasks.absent_peer_task, timeout=120)
    assert "never reached the collective" in str(err.value)
    assert time.monotonic() - t0 < 100


def test_criterion_7_collective_correctness():
    for n in _worlds():
        for verdicts in run_workers(n, _mp_tasks.collective_task).values():
            assert all(verdicts)


def test_random_payloads_bit_exact_vs_reference_ring():
    g = golden_ring()
    for n in _worlds():
        arrays = [{f"n{size}": g[f"in_N{n}_n{size}_r{r}"] for size in (1, 17, 1001, 4099)} for r in range(n)]
        results = run_workers(n, partial(_mp_tasks.random_task, arrays=arrays))
        for size in (1, 17, 1001, 4099):
            want = g[f"out_N{n}_n{size}"].view("<u4")
            for r in range(n):
                assert np.array_equal(results[r][f"n{size}"].view("<u4"), want)
                assert np.array_equal(results[r][f"n{size}_tensor"].view("<u4"), want)


def test_every_algorithm_bit_exact_over_ipc():
    """LL, one-shot and two-shot (fused and unfused) all reproduce the reference ring's bits."""
    g = golden_ring()
    for n in _worlds():
        arrays = [{f"n{size}": g[f"in_N{n}_n{size}_r{r}"] for size in (1, 17, 1001, 4099)} for r in range(n)]
        results = run_workers(n, partial(_mp_tasks.every_algorithm_task, arrays=arrays))
        for size in (1, 17, 1001, 4099):
            want = g[f"out_N{n}_n{size}"].view("<u4")
            for r in range(n):
                for variant in ("fused_ll", "fused_one", "fused_two", "fused_push", "fused_push1", "fused_ll128", "fused_ll128_1", "plain_one",
                                "plain_two", "gate_ll", "gate_two"):
                    got = results[r][f"n{size}_{variant}"].view("<u4")
                    assert np.array_equal(got, want), (n, size, r, variant)


def test_fused_algorithms_large_multirow_vs_oracle():
    from oracle import ring_oracle
    from paper_1811_11141_b200 import _native

    sizes = (4099, 16705, 40000, 65536, 131075, 262144)  # up to the LL area's 1 MB per source
    algos = (_native.ALGO_LL, _native.ALGO_ONESHOT, _native.ALGO_TWOSHOT, _native.ALGO_PUSH, _native.ALGO_PUSH_ONESHOT,
             _native.ALGO_LL128, _native.ALGO_LL128_ONESHOT)
    for n in _worlds():
        res = run_workers(n, partial(_mp_tasks.sizes_task, sizes=sizes, algos=algos))
        for size in sizes:
            want = ring_oracle.ring_allreduce([res[r][("in", size)] for r in range(n)])[0]
            for algo in algos:
                for r in range(n):
                    got = res[r][(algo, size)]
                    bad = np.flatnonzero(got.view("<u4") != want.view("<u4"))
                    assert bad.size == 0, (n, size, algo, r, bad.size, int(bad[0]))


@pytest.mark.parametrize("algo,deferred,gate", [(0, False, False), (3, False, False), (1, False, False),
                                               (2, False, False), (0, True, False), (0, False, True)])
def test_autograd_merged_sync_matches_reference_fold(algo, deferred, gate):
    from oracle import ring_oracle

    n = max(_worlds())
    results = run_workers(n, partial(_mp_tasks.autograd_task, algo=algo, deferred=deferred, gate=gate))
    assert all(results[r][2] for r in range(n)), "the test model's backward is not deterministic"
    groups = MergePlan(frozenset({2, 4}), 4).groups()
    assert groups == [(1, 2), (3, 4)]
    for low, high in groups:
        buckets = [np.concatenate([results[r][0][layer - 1].reshape(-1) for layer in range(high, low - 1, -1)])
                   for r in range(n)]
        want = ring_oracle.ring_allreduce(buckets)[0]
        for r in range(n):
            got = np.concatenate([results[r][1][layer - 1].reshape(-1) for layer in range(high, low - 1, -1)])
            bad = np.flatnonzero(got.view("<u4") != want.view("<u4"))
            if bad.size:
                i = int(bad[0])
                xs = [np.float32(b[i]) for b in buckets]
                rot = {}
                for s in range(n):
                    acc = xs[s]
                    for k in range(1, n):
                        acc = np.float32(acc + xs[(s + k) % n])
                    rot[s] = bool(acc == got[i])
                raise AssertionError(f"group {(low, high)} rank {r}: {bad.size} mismatches, first {i} "
                                     f"(of {got.size}); got {got[i]!r} want {want[i]!r}; rotations matching got: {rot}")


def test_nvls_opt_in_within_tolerance():
    """Opt-in NVLS (in-switch fp32 reduction): within N ulps of the exact sum, identical on
    every rank (scripts/nvls_check.py exits non-zero otherwise)."""
    import subprocess
    import sys

    n = max(_worlds())
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29571", "scripts/nvls_check.py"]
    proc = subprocess.run(cmd, cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    assert '"ok": true' in proc.stdout


def test_bench_local_measurement_shape():
    ms = bench_local(2, [4096, 65536, 1 << 22], repeats=3, warmups=2)
    assert [m.nbytes for m in ms] == [4096, 65536, 1 << 22]
    assert all(m.n_nodes == 2 and 0 < m.seconds < 1e-2 for m in ms)
    with pytest.raises((RuntimeError, ValueError), match="multiples of 4"):
        bench_local(2, [10], repeats=1, warmups=0)


def test_emulate_local_verified_report():
    profile = make_profile([40, 0, 24, 16], [4e-3, 3e-3, 3e-3, 2e-3], 5e-3)
    plan = MergePlan(frozenset({4}), 4)
    reports = emulate_local(2, profile, plan, 3, warmup=1)
    assert set(reports) == {0, 1}
    for r in reports.values():
        assert isinstance(r, EmulationReport) and r.verified
        assert len(r.iteration_seconds) == 3
        assert r.allreduce_count == 2 * 4
        assert set(r.group_comm_seconds) == {1, 3}
        assert r.mean_seconds >= profile.forward_time + profile.total_backward_time - 1e-4


def test_emulate_fused_and_unfused_agree():
    profile = synth_profile(30, param_range=(1e3, 3e5), time_scale=2e-3, seed=4)
    plan = MergePlan(frozenset({3, 4, 5, 10, 11, 20, 30}), 30)
    n = max(_worlds())
    for fused in (False, True):
        for graph in (False, True):
            reports = run_workers(n, partial(_mp_tasks.emulate_task, profile=profile, plan=plan, fused=fused, graph=graph))
            assert all(r.verified for r in reports.values()), (fused, graph)


def test_criterion_8_calibrate_then_predict():
    n = max(_worlds())
    sizes = [32768, 131072, 262144, 524288, 1048576, 2097152, 4194304, 8388608]
    model = fit_ab(bench_local(n, sizes, repeats=20, warmups=3))
    profile = synth_profile(8, param_range=(1e4, 2e5), time_scale=15e-3, seed=1)
    for plan in (find_merge_plan(profile, model), MergePlan(frozenset(range(2, 9)), 8)):
        predicted = simulate_mgwfbp(profile, model, plan).t_iter
        for graph in (False, True):
            reports = emulate_local(n, profile, plan, 20, warmup=2, graph=graph)
            assert all(r.verified for r in reports.values())
            measured = max(r.mean_seconds for r in reports.values())
            assert abs(measured - predicted) / predicted <= 0.05, (measured, predicted)


def test_online_replanning_from_live_spans():
    """the fused kernels' own spans refit (a, b) and re-run Algorithm 1."""
    res = run_workers(2, partial(_mp_tasks.replan_task, iterations=4))
    for r in res.values():
        assert r["verified"] and r["consistent"]
        assert r["samples"] == 4 * 54
        assert 0 <= r["a"] < 1e-3 and 0 < r["b"] < 1e-9  # µs-class startup, > 1 GB/s


def test_bf16_exchange_over_ipc_vs_oracle():
    """bf16 on the wire, fp32 accumulation, one rounding: bit-exact vs the oracle for the
    AUTO path (scale 1) and every explicit algorithm -- LL, one-shot, two-shot (scale 1/2)."""
    from oracle import ring_oracle

    sizes = (1, 17, 1001, 4099, 65543, 1 << 20)
    for n in _worlds():
        res = run_workers(n, partial(_mp_tasks.bf16_task, sizes=sizes))
        for size in sizes:
            ins = [res[r][("in", size)] for r in range(n)]
            want1 = ring_oracle.ring_allreduce_bf16(ins)
            want_half = ring_oracle.ring_allreduce_bf16(ins, scale=0.5)
            for r in range(n):
                assert np.array_equal(res[r][("auto", size)], want1), (n, size, r)
                assert np.array_equal(res[r][("one", size)], want_half), (n, size, r, "one")
                assert np.array_equal(res[r][("two", size)], want_half), (n, size, r, "two")
                assert np.array_equal(res[r][("ll128", size)], want_half), (n, size, r, "ll128")
                if size <= 131072:
                    assert np.array_equal(res[r][("ll", size)], want_half), (n, size, r, "ll")


def test_autograd_bf16_parameters():
    from oracle import ring_oracle

    n = max(_worlds())
    res = run_workers(n, _mp_tasks.autograd_bf16_task)
    for low, high in MergePlan(frozenset({2, 4}), 4).groups():
        buckets = [np.concatenate([res[r][0][layer - 1] for layer in range(high, low - 1, -1)]) for r in range(n)]
        want = ring_oracle.ring_allreduce_bf16(buckets, scale=1.0 / n)
        for r in range(n):
            got = np.concatenate([res[r][1][layer - 1] for layer in range(high, low - 1, -1)])
            assert np.array_equal(got, want), (low, high, r, int(np.count_nonzero(got != want)))


def test_randomized_stress_every_algorithm_and_dtype():
    """300 back-to-back collectives per rank with random sizes (to 2 M elements), row splits,
    dtypes and algorithms (the same sequence on every rank): exact integer results, no
    protocol error -- buffer reuse across algorithm switches is safe."""
    for n in _worlds():
        res = run_workers(n, partial(_mp_tasks.stress_task, iterations=300, seed=2024 + n), timeout=600)
        for r, (n_bad, first) in res.items():
            assert n_bad == 0, (n, r, first)


@pytest.mark.parametrize("task", ["cta_cap_mismatch_task", "swapped_groups_task", "iteration_mismatch_task",
                                  "algo_mismatch_task"])
def test_settings_disagreement_raises_fast(task):
    """Per-rank CTA caps, swapped group order, different iterations: every rank raises
    ProtocolError within a second (the collective tag in every barrier flag / LL header,
    the reference's frame header check allreduce_net.py:340-345) -- no 20 s timeout, no
    silently crossed sums."""
    results = run_workers(2, getattr(_mp_tasks, task), timeout=120)
    for rank, (seconds, err) in results.items():
        assert err is not None and ("disagree" in err or "aborted" in err), (rank, err)
        assert seconds < 1.0, (rank, seconds)


def test_threshold_disagreement_raises_fast():
    results = run_workers(2, _mp_tasks.threshold_mismatch_task, timeout=120)
    for rank, outcomes in results.items():
        for seconds, err in outcomes:
            assert err is not None and ("disagree" in err or "aborted" in err), (rank, err)
            assert seconds < 1.0, (rank, seconds)


def test_emulate_bf16_engine_verified():
    from functools import partial

    profile = resnet50_like(backward_seconds=4e-3, forward_seconds=2e-3)
    plan = find_merge_plan(profile, CommModel(a=2e-5, b=1.5e-12))
    for n in _worlds():
        res = run_workers(n, partial(_mp_tasks.emulate_bf16_task, profile=profile, plan=plan))
        for verified, count in res.values():
            assert verified
            assert count == 4 * len(plan.groups())


def test_wide_push_grid_above_threshold_vs_oracle():
    """Buckets >= 112 MiB launch the push two-shot with 512 CTAs (two waves over the 296
    resident): still bit-exact vs the oracle, fp32 (ragged rows) and bf16."""
    n32 = (112 << 20) // 4 + 12_347
    n16 = (112 << 20) // 2 + 9_001
    n = min(_worlds())
    res = run_workers(n, partial(_mp_tasks.wide_push_task, n32=n32, n16=n16), capacity_bytes=(120 << 20),
                      timeout=300.0)
    for r in range(n):
        assert res[r] == {"f32_bad": 0, "b16_bad": 0}, (r, res[r])
