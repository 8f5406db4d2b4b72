"""The C-ABI boundary on a CPU-only host: the in-tree library exists, loads, and exports
every entry point include/mgwfbp_b200.h declares.  No compute call is made here; only
argument validation that fails before CUDA is touched."""

import ctypes

import pytest

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
