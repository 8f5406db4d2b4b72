"""Profiles: validation, generators bit-identical to the reference's, new BASELINE profiles
(reference tests: /root/reference/pkg/tests/test_model_profile.py)."""

import math

import pytest

from conftest import golden_planner, make_profile
from paper_1811_11141_b200 import (
    LayerProfile,
    ModelProfile,
    bert_base_like,
    googlenet_like,
    load_profile,
    resnet50_like,
    save_profile,
    synth_profile,
    vgg16_like,
)


def test_layer_validation():
    for kw in (dict(index=0, params=1, backward_time=1e-3), dict(index=1, params=-1, backward_time=1e-3),
               dict(index=1, params=1, backward_time=-1e-3), dict(index=1, params=1, backward_time=math.nan)):
        with pytest.raises(ValueError):
            LayerProfile(**kw)
    LayerProfile(index=1, params=0, backward_time=0.0)


def test_profile_validation():
    with pytest.raises(ValueError):
        make_profile([], [], 0.1)
    with pytest.raises(ValueError):
        ModelProfile(name="x", layers=(LayerProfile(2, 1, 1e-3),), forward_time=0.1)
    with pytest.raises(ValueError):
        make_profile([1], [1e-3], -0.1)
    with pytest.raises(ValueError):
        make_profile([1], [1e-3], 0.1, element_bytes=3)
    with pytest.raises(ValueError):
        ModelProfile(name="", layers=(LayerProfile(1, 1, 1e-3),), forward_time=0.1)


def test_profile_accessors():
    p = make_profile([10, 0, 30], [1e-3, 2e-3, 3e-3], 0.05, element_bytes=8)
    assert p.num_layers == 3 and p.total_params == 40
    assert p.total_backward_time == pytest.approx(6e-3)
    assert p.param_counts() == [10, 0, 30]
    assert p.backward_times() == [1e-3, 2e-3, 3e-3]
    assert p.message_bytes(1) == 80 and p.message_bytes(2) == 0


@pytest.mark.parametrize(
    "key,build",
    [
        ("resnet50_like", lambda: resnet50_like()),
        ("resnet50_like_fast", lambda: resnet50_like(backward_seconds=0.012, forward_seconds=0.006)),
        ("googlenet_like", lambda: googlenet_like()),
        ("synth_1000", lambda: synth_profile(1000, param_range=(1024, 16_777_216), seed=0)),
        ("synth_12x5", lambda: synth_profile(12, seed=5)),
    ],
)
def test_generators_bit_identical_to_reference(key, build):
    g = golden_planner()["named"][key]
    p = build()
    assert p.name == g["name"]
    assert p.param_counts() == g["params"]
    assert p.backward_times() == g["backward_times"]  # exact float equality
    assert p.forward_time == g["forward_time"]


def test_synth_profile_deterministic_and_in_range():
    a, b, c = synth_profile(12, seed=5), synth_profile(12, seed=5), synth_profile(12, seed=6)
    assert a == b and c != a and a.name == "synth-12x5"
    assert all(1 <= l.params <= 5_500_000 and l.backward_time > 0 for l in a.layers)
    assert a.forward_time == pytest.approx(0.5 * a.total_backward_time)
    for kw in (dict(num_layers=0), dict(num_layers=4, param_range=(0.0, 10.0)), dict(num_layers=4, time_scale=-1.0)):
        with pytest.raises(ValueError):
            synth_profile(**kw)


def test_resnet50_and_googlenet_shapes():
    r = resnet50_like()
    assert r.num_layers == 54 and r.total_params == 25_503_912 and 4 * r.total_params == 102_015_648
    assert r.total_backward_time == pytest.approx(0.2) and r.forward_time == 0.1
    g = googlenet_like()
    assert g.num_layers == 64 and g.total_params == 13_365_696
    assert g.total_backward_time == pytest.approx(0.18)


def test_baseline_profiles():
    g7 = googlenet_like(aux=False)
    assert (g7.num_layers, g7.total_params) == (58, 6_990_272)
    assert g7.total_backward_time == pytest.approx(0.18)
    v = vgg16_like()
    assert (v.num_layers, v.total_params) == (16, 138_357_544)
    assert v.param_counts()[13] == 102_764_544  # fc6
    bert = bert_base_like()
    assert (bert.num_layers, bert.total_params) == (199, 109_482_240)
    assert sum(1 for l in bert.layers if l.params <= 3072) == 124
    assert bert.param_counts()[0] == 23_440_896


def test_profile_json_round_trip(tmp_path):
    p = synth_profile(9, seed=42)
    path = tmp_path / "p.profile.json"
    save_profile(p, path)
    assert load_profile(path) == p
    with open(path) as fh:
        assert load_profile(fh) == p
    with open(path, "rb") as fh:
        assert load_profile(fh) == p


def test_profile_malformed_documents(tmp_path):
    path = tmp_path / "bad.json"
    for text in ('{"name": "x", "layers": []}', "[1, 2, 3]", '{"name": "x", "forward_time": 0.1, "layers": [{"index": 1}]}'):
        path.write_text(text)
        with pytest.raises(ValueError):
            load_profile(path)
