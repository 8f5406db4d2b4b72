"""Generate the golden fixtures from the unmodified reference (run HERE only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py tests/golden

Imports the reference package as ``mgwfbp`` straight from the read-only mount
and writes:

* ``planner.json`` -- the reference's 102 archived greedy/brute-force
  counterexamples re-verified live, 300 frozen random instances (the
  reference's own ``draw_instance`` / ``draw_mixed_instance`` generators) with
  the reference's merge plans, brute-force plans and all four timelines, the
  named profiles' layer tables and plans, a criterion-6 sweep, derive/fit
  results.
* ``ring.npz`` -- per-rank fp32 inputs and the reduced output of the
  reference's real multi-process loopback-TCP ``ring_allreduce`` for
  N in {2, 3, 4, 8} at several lengths (pins the per-element fold order).

The GPU box never runs this script; it only reads the committed fixtures.
"""

from __future__ import annotations

import importlib.util
import json
import pathlib
import random
import sys
from functools import partial

import numpy as np

import mgwfbp as ref  # the reference, via PYTHONPATH=/root/reference/pkg/src

REF_TESTS = pathlib.Path("/root/reference/pkg/tests")
RING_SIZES = (1, 17, 1001, 4099)
RING_N = (2, 3, 4, 8)


def _ref_conftest():
    spec = importlib.util.spec_from_file_location("ref_conftest", REF_TESTS / "conftest.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _timeline(tl) -> dict:
    return {
        "tau_c": list(tl.tau_c),
        "t_c": list(tl.t_c),
        "comm_end": list(tl.comm_end),
        "t_iter": tl.t_iter,
        "compute_time": tl.compute_time,
        "t_c_no": tl.t_c_no,
        "case": tl.case.value,
    }


def _instance(profile, model) -> dict:
    return {
        "params": profile.param_counts(),
        "backward_times": profile.backward_times(),
        "forward_time": profile.forward_time,
        "element_bytes": profile.element_bytes,
        "a": model.a,
        "b": model.b,
    }


def _solve(profile, model, brute: bool) -> dict:
    plan = ref.find_merge_plan(profile, model)
    out = {
        "plan": sorted(plan.merged_layers),
        "naive": _timeline(ref.simulate_naive(profile, model)),
        "wfbp": _timeline(ref.simulate_wfbp(profile, model)),
        "synceasgd": _timeline(ref.simulate_sync_easgd(profile, model)),
        "mgwfbp": _timeline(ref.simulate_mgwfbp(profile, model, plan)),
        "groups": [list(g) for g in plan.groups()],
    }
    if brute:
        out["brute_plan"] = sorted(ref.brute_force_plan(profile, model).merged_layers)
    return out


def planner_fixture() -> dict:
    conf = _ref_conftest()
    doc: dict = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src/mgwfbp"}

    archive = json.loads((REF_TESTS / "artifacts" / "planner_oracle_counterexamples.json").read_text())
    cases = []
    for m in archive["mismatches"]:
        profile = conf.make_profile(m["params"], m["backward_times"], m["forward_time"], m["element_bytes"])
        model = ref.CommModel(m["a"], m["b"])
        live = ref.find_merge_plan(profile, model)
        assert sorted(live.merged_layers) == m["greedy_plan"], "archive no longer reproduces"
        assert ref.simulate_mgwfbp(profile, model, live).t_iter == m["greedy_t_iter"]
        entry = {k: m[k] for k in ("index", "params", "backward_times", "forward_time", "element_bytes", "a", "b",
                                    "greedy_plan", "oracle_plan", "greedy_t_iter", "oracle_t_iter")}
        entry["wfbp_t_iter"] = ref.simulate_wfbp(profile, model).t_iter
        entry["synceasgd_t_iter"] = ref.simulate_sync_easgd(profile, model).t_iter
        cases.append(entry)
    doc["archive"] = {"seed": archive["seed"], "instances": archive["instances"], "cases": cases}

    rnd = []
    rng = random.Random(20261018)
    for k in range(300):
        max_layers = (12, 12, 24, 60)[k % 4]
        if k % 3 == 2:
            profile, model = conf.draw_mixed_instance(rng, max_layers)
        else:
            profile, model = conf.draw_instance(rng, max_layers)
        entry = _instance(profile, model)
        entry.update(_solve(profile, model, brute=profile.num_layers <= 10))
        rnd.append(entry)
    doc["random"] = rnd

    named = {}
    for key, prof in (
        ("resnet50_like", ref.resnet50_like()),
        ("resnet50_like_fast", ref.resnet50_like(backward_seconds=0.012, forward_seconds=0.006)),
        ("googlenet_like", ref.googlenet_like()),
        ("synth_1000", ref.synth_profile(1000, param_range=(1024, 16_777_216), seed=0)),
        ("synth_12x5", ref.synth_profile(12, seed=5)),
    ):
        rows = {
            "name": prof.name,
            "forward_time": prof.forward_time,
            "params": prof.param_counts(),
            "backward_times": prof.backward_times(),
            "plans": [],
        }
        for a, b in ((1.5e-5, 1.4e-12), (1e-4, 1e-10), (1e-3, 1e-9), (45.26e-6 * 14, 8e-10)):
            model = ref.CommModel(a, b)
            plan = ref.find_merge_plan(prof, model)
            rows["plans"].append({
                "a": a,
                "b": b,
                "plan": sorted(plan.merged_layers),
                "mgwfbp_t_iter": ref.simulate_mgwfbp(prof, model, plan).t_iter,
                "wfbp_t_iter": ref.simulate_wfbp(prof, model).t_iter,
                "synceasgd_t_iter": ref.simulate_sync_easgd(prof, model).t_iter,
            })
        named[key] = rows
    doc["named"] = named

    params = ref.CollectiveParams(ref.Collective.RING, 4, 45.26e-6, 8e-10, 5e-11)
    res = ref.sweep(ref.resnet50_like(), params, [4, 8, 16, 32, 64])
    doc["sweep_resnet50_ring"] = {
        "rows": [[r.n_nodes, r.strategy.value, r.t_iter, r.speedup, r.t_c_no] for r in res.rows],
        "crossing": ref.crossing_node_count(res),
    }
    frozen = ref.sweep(ref.resnet50_like(), params, [4, 64], [ref.Strategy.MGWFBP], freeze_plan=True)
    doc["sweep_frozen"] = [[r.n_nodes, r.strategy.value, r.t_iter, r.speedup, r.t_c_no] for r in frozen.rows]

    derive = []
    for alg in ref.Collective:
        for n in (2, 4, 8, 64):
            m = ref.derive_ab(ref.CollectiveParams(alg, n, 45.26e-6, 8e-10, 5e-11))
            derive.append([alg.value, n, m.a, m.b])
    doc["derive_ab"] = derive
    rng = random.Random(7)
    samples = [ref.Measurement(1 << k, (3e-4 + 2e-9 * (1 << k)) * (1 + rng.uniform(-0.02, 0.02)), 4)
               for k in range(12, 24) for _ in range(3)]
    fit = ref.fit_ab(samples)
    doc["fit_ab"] = {"samples": [[s.nbytes, s.seconds, s.n_nodes] for s in samples], "a": fit.a, "b": fit.b}
    return doc


def _ring_task(config, session, *, sizes):
    """Run in every spawned reference worker: reduce seeded N(0,1) fp32 data."""
    out = {}
    for n in sizes:
        vals = np.random.default_rng(1000 + config.rank).standard_normal(n).astype("<f4")
        buf = ref.GradientBuffer(1, 1, vals.copy())
        ref.ring_allreduce(buf, config, session)
        out[n] = (vals, buf.values.copy())
    return out


def ring_fixture() -> dict:
    arrays = {}
    for n_ranks in RING_N:
        results = ref.run_workers(n_ranks, partial(_ring_task, sizes=RING_SIZES))
        for n in RING_SIZES:
            reduced = results[0][n][1]
            for r in range(n_ranks):
                arrays[f"in_N{n_ranks}_n{n}_r{r}"] = results[r][n][0]
                assert np.array_equal(results[r][n][1].view("<u4"), reduced.view("<u4")), "ranks disagree"
            arrays[f"out_N{n_ranks}_n{n}"] = reduced
    return arrays


def main(outdir: str) -> None:
    out = pathlib.Path(outdir)
    out.mkdir(parents=True, exist_ok=True)
    doc = planner_fixture()
    (out / "planner.json").write_text(json.dumps(doc) + "\n")
    np.savez_compressed(out / "ring.npz", **ring_fixture())
    print(f"wrote {out / 'planner.json'} and {out / 'ring.npz'}")


if __name__ == "__main__":
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
    main(sys.argv[1] if len(sys.argv) > 1 else str(pathlib.Path(__file__).resolve().parent))
