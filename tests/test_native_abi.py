"""The C-ABI boundary on a CPU-only host: the in-tree library exists, loads, and exports
every entry point include/mgwfbp_b200.h declares.  No compute call is made here; only
argument validation that fails before CUDA is touched."""

import ctypes

import pytest

from conftest import ROOT
from paper_1811_11141_b200 import _native


def test_header_declares_the_expected_surface():
    names = _native.declared_symbols()
    for required in ("mgw_pack", "mgw_unpack", "mgw_allreduce", "mgw_comm_create", "mgw_comm_open_peers",
                     "mgw_spin_ns", "mgw_sched_create", "mgw_sched_run", "mgw_last_error"):
        assert required in names
    assert set(names) == set(_native._SIGNATURES)


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.lib()
    for name in _native.declared_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.mgw_version()


def test_library_is_built_for_sm100a():
    data = _native.library_path().read_bytes()
    assert b"sm_100a" in data


def test_invalid_arguments_map_to_value_error_before_cuda():
    handle = ctypes.c_void_p()
    with pytest.raises(ValueError):
        _native.call("mgw_comm_create", 0, 0, 0, 1024, ctypes.byref(handle), None)
    with pytest.raises(ValueError):
        _native.call("mgw_comm_create", 3, 2, 0, 1024, ctypes.byref(handle), None)
    with pytest.raises(ValueError):
        _native.call("mgw_spin_ns", -1, None)
    with pytest.raises(ValueError):
        _native.call("mgw_allreduce", None, 16, 0, None)
    assert "comm is null" in _native.last_error()


def test_status_codes_map_to_reference_exceptions():
    _native.check(0)
    with pytest.raises(ValueError):
        _native.check(1)
    with pytest.raises(_native.ProtocolError):
        _native.check(2)
    with pytest.raises(RuntimeError):
        _native.check(3)
    assert issubclass(_native.ProtocolError, RuntimeError)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setenv("MGWFBP_B200_LIB", str(tmp_path / "absent.so"))
    with pytest.raises(RuntimeError, match="native data path missing"):
        _native.lib()


def _tag(group, n, kind, grid, scale=1.0):
    out = ctypes.c_uint32()
    _native.call("mgw_debug_collective_tag", group, n, kind, grid, ctypes.c_float(scale), ctypes.byref(out))
    return out.value


def test_collective_tag_separates_every_field():
    """The 32-bit tag in every barrier flag / LL header (the reference's frame header check,
    allreduce_net.py:340-345) changes with each thing ranks must agree on: length (also
    beyond 2^32), kernel family incl. dtype (kinds 1..11), grid, scale and group tag."""
    base = _tag(7, 100_000, 3, 98)
    variants = {
        "length": _tag(7, 100_001, 3, 98),
        "length_2^32": _tag(7, 100_000 + (1 << 32), 3, 98),
        "grid": _tag(7, 100_000, 3, 97),
        "scale": _tag(7, 100_000, 3, 98, 0.5),
        "group": _tag(8, 100_000, 3, 98),
    }
    for kind in range(1, 12):
        if kind != 3:
            variants[f"kind{kind}"] = _tag(7, 100_000, kind, 98)
    assert base == _tag(7, 100_000, 3, 98)  # deterministic: every rank computes the same
    for name, t in variants.items():
        assert t != base, name
    assert len(set(variants.values())) == len(variants)


def test_group_tag_mixes_layer_and_iteration():
    from paper_1811_11141_b200.allreduce_net import group_tag

    tags = {group_tag(low, it) for low in range(1, 60) for it in range(0, 50)}
    assert len(tags) == 59 * 50
    assert all(0 <= t < 1 << 32 for t in tags)


def test_python_constants_match_the_header():
    """Every MGW_ALGO_* / MGW_SCHED_* / MGW_OPT_* / MGW_DEV_* / status code the header
    defines has the same value in _native (the ctypes binding a reference user imports)."""
    import re

    from paper_1811_11141_b200 import _native

    header = (ROOT / "include" / "mgwfbp_b200.h").read_text()
    defs = dict(re.findall(r"#define (MGW_[A-Z0-9_]+) (\d+)u?\b", header))
    prefixes = {"MGW_ALGO_": "ALGO_", "MGW_SCHED_": "SCHED_", "MGW_OPT_": "OPT_", "MGW_DEV_": "DEV_"}
    checked = 0
    for name, value in defs.items():
        for cprefix, pyprefix in prefixes.items():
            if name.startswith(cprefix):
                py = pyprefix + name[len(cprefix):]
                assert hasattr(_native, py), py
                assert getattr(_native, py) == int(value), (name, value, getattr(_native, py))
                checked += 1
    for name in ("MGW_OK", "MGW_EINVAL", "MGW_EPROTO", "MGW_ECUDA"):
        assert getattr(_native, name) == int(defs[name]), name
    assert checked >= 20
