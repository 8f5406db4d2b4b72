"""ORACLE (test infrastructure): the reference ring all-reduce and bucket layout on the CPU.

Restates, step for step:

* ``segments``           <- allreduce_net.py:360-367 (``_segments``)
* ``ring_allreduce``     <- allreduce_net.py:370-411: N-1 reduce-scatter rounds in
                            which rank r sends segment (r-k) mod N to its right
                            neighbour and adds the incoming segment (r-k-1) mod N
                            (``seg += incoming``, :401), then N-1 all-gather rounds
                            (send (r+1-k), receive and overwrite (r-k), :410).  Every
                            round's message is a snapshot taken before the round,
                            exactly as the socket exchange delivers it.
* ``pack_group``         <- allreduce_net.py:499-509 (layer ``high`` at offset 0,
                            walking down to ``low``) and :546 (per-layer slice fill)
* ``emulation_expected`` <- allreduce_net.py:507
* ``ring_allreduce_bf16`` (extension; no reference counterpart): bf16
                            inputs upcast exactly to fp32, the reference ring above
                            (same fold order), times ``scale`` when != 1, rounded once
                            to bf16 (round-to-nearest-even; ``bf16_round`` is pinned
                            against torch's fp32 -> bf16 cast in tests/test_oracle.py)

A C build of the same ring (``ring_oracle.c`` -> ``_build/libring_oracle.so``,
one thread per simulated rank) is used when present; ``tests/test_oracle.py``
checks both against the reference-generated golden vectors.
"""

from __future__ import annotations

import ctypes
import pathlib

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libring_oracle.so"
_lib = None


def segments(n_elements: int, n_parts: int) -> tuple[list[int], list[int]]:
    q, r = divmod(n_elements, n_parts)
    sizes = [q + 1 if i < r else q for i in range(n_parts)]
    offsets = [0] * n_parts
    for i in range(1, n_parts):
        offsets[i] = offsets[i - 1] + sizes[i - 1]
    return sizes, offsets


def ring_allreduce_numpy(rank_values) -> list[np.ndarray]:
    """All ranks' buffers after the reference ring (pure numpy, lock-step)."""
    bufs = [np.array(v, dtype="<f4", copy=True) for v in rank_values]
    n_ranks = len(bufs)
    n = len(bufs[0])
    if any(len(b) != n for b in bufs):
        raise ValueError("ranks disagree on the buffer length")
    sizes, offsets = segments(n, n_ranks)

    def seg(buf, idx):
        return buf[offsets[idx] : offsets[idx] + sizes[idx]]

    for step in range(n_ranks - 1):
        outgoing = [seg(bufs[r], (r - step) % n_ranks).copy() for r in range(n_ranks)]
        for r in range(n_ranks):
            recv_idx = (r - step - 1) % n_ranks
            target = seg(bufs[r], recv_idx)
            target += outgoing[(r - 1) % n_ranks]
    for step in range(n_ranks - 1):
        outgoing = [seg(bufs[r], (r + 1 - step) % n_ranks).copy() for r in range(n_ranks)]
        for r in range(n_ranks):
            recv_idx = (r - step) % n_ranks
            seg(bufs[r], recv_idx)[:] = outgoing[(r - 1) % n_ranks]
    return bufs


def _load():
    global _lib
    if _lib is None and _SO.exists():
        lib = ctypes.CDLL(str(_SO))
        lib.oracle_ring_allreduce.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        lib.oracle_ring_allreduce.restype = ctypes.c_int
        lib.oracle_pack.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                                    ctypes.c_void_p]
        lib.oracle_pack.restype = None
        _lib = lib
    return _lib


def have_c() -> bool:
    return _load() is not None


def ring_allreduce_c(rank_values, threads: int | None = None) -> list[np.ndarray]:
    """Same ring in C, one pthread per simulated rank (``threads=1``: lock-step loop)."""
    lib = _load()
    if lib is None:
        raise RuntimeError(f"C oracle not built ({_SO}); run `make -C oracle`")
    bufs = [np.array(v, dtype="<f4", copy=True) for v in rank_values]
    n = len(bufs[0])
    if any(len(b) != n for b in bufs):
        raise ValueError("ranks disagree on the buffer length")
    ptrs = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    rc = lib.oracle_ring_allreduce(ptrs, len(bufs), n, len(bufs) if threads is None else threads)
    if rc != 0:
        raise RuntimeError(f"oracle_ring_allreduce failed ({rc})")
    return bufs


def ring_allreduce(rank_values) -> list[np.ndarray]:
    return ring_allreduce_c(rank_values) if have_c() else ring_allreduce_numpy(rank_values)


def group_rows(counts, low: int, high: int) -> list[tuple[int, int, int]]:
    """``(layer, params, offset)`` rows of one group bucket, layer ``high`` first."""
    rows, off = [], 0
    for layer in range(high, low - 1, -1):
        p = counts[layer - 1]
        rows.append((layer, p, off))
        off += p
    return rows


def pack_group(layer_values: dict, counts, low: int, high: int, scale: float = 1.0) -> np.ndarray:
    rows = group_rows(counts, low, high)
    total = sum(p for _, p, _ in rows)
    bucket = np.empty(total, dtype="<f4")
    for layer, p, off in rows:
        if p:
            part = np.asarray(layer_values[layer], dtype="<f4")
            bucket[off : off + p] = part if scale == 1.0 else part * np.float32(scale)
    return bucket


def unpack_group(bucket: np.ndarray, counts, low: int, high: int) -> dict:
    return {layer: bucket[off : off + p].copy() for layer, p, off in group_rows(counts, low, high) if p}


def emulation_expected(n_workers: int, layer: int) -> float:
    return float(n_workers * (n_workers + 1) // 2 + n_workers * (layer % 5))


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float32, exact."""
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest even (NaN stays a quiet NaN)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    if nan.any():
        r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def ring_allreduce_bf16(rank_values_u16, scale: float = 1.0) -> np.ndarray:
    """bf16 gradients with fp32 accumulation: the reference fold over upcast inputs,
    scaled (fp32, only when ``scale != 1``) and rounded once.  Same bits on every rank."""
    acc = ring_allreduce([bf16_to_f32(v) for v in rank_values_u16])[0]
    if scale != 1.0:
        acc = (acc * np.float32(scale)).astype(np.float32)
    return bf16_round(acc)
