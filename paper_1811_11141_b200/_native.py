"""ctypes binding of the C ABI in ``include/mgwfbp_b200.h``.

The shared library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_1811_11141_b200.build``) into ``_lib/libmgwfbp_b200.so``.
There is deliberately no fallback: if the library is missing or CUDA is not
usable, every data-path call raises.  Status codes map to exceptions exactly as
the header documents: 1 -> ValueError, 2 -> ProtocolError, 3 -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

LIB_DIR = pathlib.Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / "libmgwfbp_b200.so"

MGW_OK, MGW_EINVAL, MGW_EPROTO, MGW_ECUDA = 0, 1, 2, 3
(ALGO_AUTO, ALGO_ONESHOT, ALGO_TWOSHOT, ALGO_LL, ALGO_NVLS, ALGO_PUSH, ALGO_PUSH_ONESHOT, ALGO_PUSH_PIPE,
 ALGO_LL128, ALGO_LL128_ONESHOT) = range(10)
SCHED_FILL, SCHED_GRAPH, SCHED_HOSTIO, SCHED_FUSED, SCHED_PDL, SCHED_BF16 = 1, 2, 4, 8, 16, 32
OPT_WIDE_MIN_BYTES = 4  # mgw_set_option key: push two-shot buckets >= this launch 512 CTAs (0 = off)
OPT_LOCAL_MIN_SLOTS = 3  # mgw_set_option key: single-rank group kernel minimum slots per CTA
OPT_PIPE_SUB_SLOTS = 2  # mgw_set_option key: pipelined two-shot sub-chunk slots per part
OPT_ROWS_PATH = 1  # mgw_set_option key: 0 auto, 1 LDG only, 2 TMA bulk wherever allowed
TIME_GRAPH = 256  # mgw_time_exchange: replay the reps as one CUDA graph
DEV_OK, DEV_MISMATCH, DEV_TIMEOUT, DEV_PEER_ABORT = 0, 1, 2, 3
DEV_LENGTH_MISMATCH = DEV_MISMATCH  # round-1 name
IPC_HANDLE_BYTES = 64
MAX_RANKS = 8


class ProtocolError(RuntimeError):
    """Peer-level disagreement: length mismatch, dead/absent peer, timeout
    (reference: allreduce_net.py:57-58)."""


class TensorDesc(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("count", ctypes.c_int64), ("offset", ctypes.c_int64)]


class Group(ctypes.Structure):
    _fields_ = [
        ("head_layer", ctypes.c_int32),
        ("desc_begin", ctypes.c_int32),
        ("desc_count", ctypes.c_int32),
        ("algo", ctypes.c_int32),
        ("n_elem", ctypes.c_int64),
        ("ready_ns", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SIGNATURES = {
    "mgw_version": ([], ctypes.c_char_p),
    "mgw_last_error": ([ctypes.c_char_p, ctypes.c_size_t], _I),
    "mgw_device_count": ([ctypes.POINTER(_I)], _I),
    "mgw_spin_ns": ([_I64, _P], _I),
    "mgw_desc_upload": ([ctypes.POINTER(TensorDesc), _I, ctypes.POINTER(_P)], _I),
    "mgw_desc_free": ([_P], _I),
    "mgw_pack": ([_P, _I, _P, _I64, ctypes.c_float, _P], _I),
    "mgw_unpack": ([_P, _I, _P, _I64, _P], _I),
    "mgw_fill_const": ([_P, _I, _P, _P], _I),
    "mgw_check_const": ([_P, _I, _P, ctypes.POINTER(_I64), _P], _I),
    "mgw_comm_create": ([_I, _I, _I, _I64, ctypes.POINTER(_P), ctypes.c_char_p], _I),
    "mgw_comm_open_peers": ([_P, ctypes.c_char_p], _I),
    "mgw_comm_destroy": ([_P], _I),
    "mgw_comm_set_timeout_ms": ([_P, _I64], _I),
    "mgw_comm_set_oneshot_max": ([_P, _I64], _I),
    "mgw_comm_set_max_ctas": ([_P, _I], _I),
    "mgw_comm_set_ll_max": ([_P, _I64], _I),
    "mgw_comm_set_gate": ([_P, _I], _I),
    "mgw_comm_set_tuning": ([_P, _I, _I64], _I),
    "mgw_comm_set_group_tag": ([_P, ctypes.c_uint32], _I),
    "mgw_comm_pick_algo": ([_P, _I64, _I, ctypes.POINTER(_I)], _I),
    "mgw_comm_clear_error": ([_P], _I),
    "mgw_comm_create_local": ([_I, _I, _I64, ctypes.POINTER(_P)], _I),
    "mgw_group_allreduce_fused": ([ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_I64),
                                   ctypes.POINTER(ctypes.c_float), _I, _I, _I, _P], _I),
    "mgw_set_option": ([_I, _I64], _I),
    "mgw_checked_violations": ([_I, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(_I)], _I),
    "mgw_debug_collective_tag": ([ctypes.c_uint32, _I64, _I, _I, ctypes.c_float, ctypes.POINTER(ctypes.c_uint32)], _I),
    "mgw_comm_input": ([_P, ctypes.POINTER(_P)], _I),
    "mgw_comm_result": ([_P, ctypes.POINTER(_P)], _I),
    "mgw_comm_pack": ([_P, _P, _I, _I64, ctypes.c_float, _P], _I),
    "mgw_allreduce": ([_P, _I64, _I, _P], _I),
    "mgw_allreduce_fused": ([_P, _P, _I, _I64, ctypes.c_float, _I, _P], _I),
    "mgw_nvls_supported": ([_I, ctypes.POINTER(_I)], _I),
    "mgw_nvls_create": ([_P, _I64, ctypes.POINTER(_I)], _I),
    "mgw_nvls_import": ([_P, _I, _I64], _I),
    "mgw_nvls_add_device": ([_P], _I),
    "mgw_nvls_bind": ([_P], _I),
    "mgw_comm_set_nvls_min": ([_P, _I64], _I),
    "mgw_group_launch": ([_P, _P, _I, _I64, ctypes.c_float, _I, _P, _P, _P], _I),
    "mgw_group_launch_bf16": ([_P, _P, _I, _I64, ctypes.c_float, _I, _P, _P, _P], _I),
    "mgw_probe_phases": ([_P, _P, _I, _I64, _I, _I, ctypes.POINTER(ctypes.c_uint64), _P], _I),
    "mgw_allreduce_fused_bf16": ([_P, _P, _I, _I64, ctypes.c_float, _I, _P], _I),
    "mgw_allreduce_fused_bf16_emulated": ([ctypes.POINTER(_P), ctypes.POINTER(_P), _I, _I64, ctypes.c_float, _I, _P],
                                          _I),
    "mgw_event_create": ([ctypes.POINTER(_P)], _I),
    "mgw_event_destroy": ([_P], _I),
    "mgw_allreduce_fused_emulated": ([ctypes.POINTER(_P), ctypes.POINTER(_P), _I, _I64, ctypes.c_float, _I, _P], _I),
    "mgw_comm_error": ([_P, ctypes.POINTER(_I)], _I),
    "mgw_comm_calls": ([_P, ctypes.POINTER(_I64)], _I),
    "mgw_time_exchange": ([_P, _P, _I, _I64, _P, _I, _I, _I, _I, ctypes.POINTER(ctypes.c_double), _P], _I),
    "mgw_allreduce_emulated": ([ctypes.POINTER(_P), ctypes.POINTER(_P), _I, _I64, _I, _P], _I),
    "mgw_sched_create": (
        [_P, ctypes.POINTER(TensorDesc), _I, ctypes.POINTER(Group), _I, ctypes.c_float, ctypes.c_uint32,
         ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P)],
        _I,
    ),
    "mgw_sched_run": ([_P, _P, _P], _I),
    "mgw_sched_times": ([_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], _I),
    "mgw_sched_kernel_times": ([_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], _I),
    "mgw_sched_events": ([_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(ctypes.c_double)], _I),
    "mgw_sched_launches": ([_P, ctypes.POINTER(_I)], _I),
    "mgw_sched_destroy": ([_P], _I),
}

_lock = threading.Lock()
_lib = None


def library_path() -> pathlib.Path:
    override = os.environ.get("MGWFBP_B200_LIB")
    return pathlib.Path(override) if override else LIB_PATH


def lib() -> ctypes.CDLL:
    """Load the native library once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = library_path()
            if not path.exists():
                raise RuntimeError(
                    f"native data path missing: {path} not built "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'` at the repo root)"
                )
            handle = ctypes.CDLL(str(path))
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = res
            _lib = handle
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().mgw_last_error(buf, len(buf))
    return buf.value.decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    if rc == MGW_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == MGW_EINVAL:
        raise ValueError(msg)
    if rc == MGW_EPROTO:
        raise ProtocolError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def declared_symbols(header: pathlib.Path | None = None) -> list[str]:
    """Function names declared in include/mgwfbp_b200.h (for the export test)."""
    import re

    header = header or pathlib.Path(__file__).resolve().parents[1] / "include" / "mgwfbp_b200.h"
    text = header.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(mgw_\w+)\s*\(", text, re.M)))


def desc_array(rows) -> ctypes.Array:
    arr = (TensorDesc * max(1, len(rows)))()
    for k, (ptr, count, offset) in enumerate(rows):
        arr[k].ptr = ptr
        arr[k].count = count
        arr[k].offset = offset
    return arr


class DeviceTable:
    """Device-resident descriptor table (uploaded once, freed with the owner)."""

    def __init__(self, rows):
        self.n = len(rows)
        self.extent = rows[-1][2] + rows[-1][1] if rows else 0
        handle = ctypes.c_void_p()
        call("mgw_desc_upload", desc_array(rows), self.n, ctypes.byref(handle))
        self.ptr = handle.value

    def close(self) -> None:
        if self.ptr:
            lib().mgw_desc_free(self.ptr)
            self.ptr = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass
