"""Shared builders and markers.

``gpu``-marked tests need a B200 (run on the GPU box with ``-m gpu``); every
other test runs on the CPU.  The instance generators restate the reference
suite's frozen generators (``/root/reference/pkg/tests/conftest.py:33-100``)
call for call, so seeded streams reproduce the reference's instances.
"""

from __future__ import annotations

import json
import math
import pathlib
import random
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1811_11141_b200 import CommModel, LayerProfile, ModelProfile  # noqa: E402

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
ACCEPTANCE_SEED = 20260818


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")
    # the in-tree libraries are build products (git-ignored): build them once on a fresh
    # checkout (nvcc cross-compiles sm_100a without a GPU), so the ABI tests see them
    lib = ROOT / "paper_1811_11141_b200" / "_lib" / "libmgwfbp_b200.so"
    oracle_lib = ROOT / "oracle" / "_build" / "libring_oracle.so"
    if not lib.exists() or not oracle_lib.exists():
        import __graft_entry__

        __graft_entry__.build()


def log_uniform(rng: random.Random, lo: float, hi: float) -> float:
    return math.exp(rng.uniform(math.log(lo), math.log(hi)))


def make_profile(params, t_b, t_f, element_bytes=4, name="case") -> ModelProfile:
    layers = tuple(LayerProfile(index=i + 1, params=p, backward_time=t) for i, (p, t) in enumerate(zip(params, t_b)))
    return ModelProfile(name=name, layers=layers, forward_time=t_f, element_bytes=element_bytes)


def draw_instance(rng: random.Random, max_layers: int = 12):
    n = rng.randint(2, max_layers)
    params = [max(1, round(log_uniform(rng, 1e2, 5e6))) for _ in range(n)]
    t_b = [log_uniform(rng, 1e-4, 2e-2) for _ in range(n)]
    t_f = log_uniform(rng, 1e-3, 5e-2)
    profile = make_profile(params, t_b, t_f, name=f"rand-{n}")
    return profile, CommModel(a=log_uniform(rng, 1e-6, 1e-2), b=log_uniform(rng, 1e-10, 1e-8))


def draw_mixed_instance(rng: random.Random, max_layers: int = 12):
    profile, model = draw_instance(rng, max_layers)
    params = [0 if rng.random() < 0.25 else p for p in profile.param_counts()]
    if sum(params) == 0:
        params[rng.randrange(len(params))] = 1000
    return make_profile(params, profile.backward_times(), profile.forward_time), model


def worked_instance():
    """t_f=4, four layers of t_b=2, messages of 1.5 + 0.25*4 = 2.5 s: naive 22,
    WFBP 16, single message 17.5, merging layer 2 gives 15.5."""
    return make_profile([1, 1, 1, 1], [2.0] * 4, 4.0, name="worked-4"), CommModel(a=1.5, b=0.25)


GREEDY_GAP_WITNESS = dict(
    params=[12855, 221, 596, 2428895, 3315117],
    t_b=[0.002519027849492765, 0.001506512706693733, 0.0006124641463250938, 0.0009339864222867493,
         0.0001508714477365246],
    t_f=0.008874705779014651,
    a=0.0023296062054062156,
    b=4.332181912040887e-09,
)


def greedy_gap_instance():
    w = GREEDY_GAP_WITNESS
    return make_profile(w["params"], w["t_b"], w["t_f"], name="greedy-gap"), CommModel(a=w["a"], b=w["b"])


_cache: dict = {}


def golden_planner() -> dict:
    if "planner" not in _cache:
        _cache["planner"] = json.loads((GOLDEN / "planner.json").read_text())
    return _cache["planner"]


def golden_ring():
    import numpy as np

    if "ring" not in _cache:
        _cache["ring"] = dict(np.load(GOLDEN / "ring.npz"))
    return _cache["ring"]


def cuda_devices() -> int:
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture
def need_gpu():
    if cuda_devices() < 1:
        pytest.skip("needs a CUDA device")


@pytest.fixture
def need_two_gpus():
    if cuda_devices() < 2:
        pytest.skip("needs >= 2 CUDA devices (one process per GPU)")


@pytest.fixture(scope="session", autouse=True)
def _checked_build_violations():
    """With the bounds-checked library (MGWFBP_B200_LIB=..._checked.so), every index the
    kernels computed during the session must have been inside its extent."""
    yield
    import ctypes
    import os

    if "checked" not in os.environ.get("MGWFBP_B200_LIB", ""):
        return
    from paper_1811_11141_b200 import _native

    if _native._lib is None:
        return
    total, checked = ctypes.c_uint64(), ctypes.c_int()
    _native.call("mgw_checked_violations", 0, ctypes.byref(total), ctypes.byref(checked))
    print(f"\nchecked build: {total.value} index violations (checked={checked.value})")
    assert checked.value == 1 and total.value == 0, f"{total.value} index violations in the checked build"
