"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the PaREM hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1412_1741_b200``) never imports it and shares no code with it.

* :func:`walk` -- the plain sequential DFA definition (oracle.c).
* :func:`states_at` -- states at given offsets (soundness checks: boundary state in R_i).
* :func:`route_stats` -- the paper's R_i = S n L counts for a given partition.
* :mod:`oracle.alg1` -- a tiny pure-Python model of Algorithm 1 that pins
  Table II and the "calculations" arithmetic; not the parity authority.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import NamedTuple

import numpy as np

DEAD = 0xFFFFFFFF
OK, EINVAL, ESYMBOL = 0, -1, -2

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _Res(C.Structure):
    _fields_ = [("match_count", C.c_uint64), ("final_state", C.c_uint32), ("accepted", C.c_uint32),
                ("bad_offset", C.c_uint64), ("status", C.c_int32), ("reserved", C.c_uint32)]


class Result(NamedTuple):
    final_state: int
    accepted: bool
    match_count: int
    status: int = OK
    bad_offset: int = 0


def lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(so):
            import buildlib

            buildlib.build_oracle()
        L = C.CDLL(so)
        u64, u32, p = C.c_uint64, C.c_uint32, C.c_void_p
        L.oracle_walk.restype = C.c_int
        L.oracle_walk.argtypes = [u32, u32, p, u32, u32, p, p, u64, C.POINTER(_Res)]
        L.oracle_states_at.restype = C.c_int
        L.oracle_states_at.argtypes = [u32, u32, p, u32, u32, p, u64, p, u64, p]
        L.oracle_lookback_stats.restype = C.c_int
        L.oracle_lookback_stats.argtypes = [u32, u32, p, u32, p, u64, p, u64, u64, C.POINTER(u64), C.POINTER(u64), p]
        L.oracle_positions.restype = C.c_int
        L.oracle_positions.argtypes = [u32, u32, p, u32, u32, p, p, u64, p, u64, C.POINTER(u64)]
        L.oracle_route_stats.restype = C.c_int
        L.oracle_route_stats.argtypes = [u32, u32, p, u32, p, u64, p, u64,
                                         C.POINTER(u64), C.POINTER(u64), p]
        _LIB = L
    return _LIB


def _tab(table) -> np.ndarray:
    t = np.ascontiguousarray(table)
    if t.dtype not in (np.uint16, np.uint32) or t.ndim != 2:
        raise ValueError("table must be a 2-D uint16/uint32 array (Q, A)")
    return t


def _bytes(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint8))


def _bitmap(accept, Q: int) -> np.ndarray:
    a = np.asarray(accept)
    if a.dtype == bool:  # bool[Q] flags
        assert a.size == Q
        return np.packbits(a, bitorder="little")
    assert a.dtype == np.uint8 and a.size == (Q + 7) // 8  # already an LSB-first bitmap
    return np.ascontiguousarray(a)


def walk(table, start: int, accept, text) -> Result:
    """Sequential DFA walk.  ``accept`` is a bool[Q] array (or an LSB-first bitmap)."""
    t = _tab(table)
    Q, A = t.shape
    T = _bytes(text)
    bm = _bitmap(accept, Q)
    r = _Res()
    lib().oracle_walk(Q, A, t.ctypes.data, t.itemsize, start, bm.ctypes.data,
                      T.ctypes.data if T.size else None, T.size, C.byref(r))
    return Result(r.final_state, bool(r.accepted), r.match_count, r.status, r.bad_offset)


def positions(table, start: int, accept, text, cap: int | None = None) -> tuple[np.ndarray, int]:
    """Match end offsets (every k with q_{k+1} in F, ascending) and their total count."""
    t = _tab(table)
    Q, A = t.shape
    T = _bytes(text)
    bm = _bitmap(accept, Q)
    cap = T.size if cap is None else cap
    out = np.empty(max(1, cap), dtype=np.uint64)
    cnt = C.c_uint64()
    rc = lib().oracle_positions(Q, A, t.ctypes.data, t.itemsize, start, bm.ctypes.data,
                                T.ctypes.data if T.size else None, T.size, out.ctypes.data, cap, C.byref(cnt))
    if rc != OK:
        raise ValueError(f"oracle_positions failed ({rc})")
    return out[: min(cap, cnt.value)], int(cnt.value)


def states_at(table, start: int, text, offsets) -> np.ndarray:
    t = _tab(table)
    Q, A = t.shape
    T = _bytes(text)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
    out = np.empty(off.size, dtype=np.uint32)
    rc = lib().oracle_states_at(Q, A, t.ctypes.data, t.itemsize, start, T.ctypes.data if T.size else None,
                                T.size, off.ctypes.data, off.size, out.ctypes.data)
    if rc != OK:
        raise ValueError(f"oracle_states_at failed ({rc})")
    return out


def route_stats(table, text, boundaries) -> tuple[int, int]:
    """(routes, route_steps) of the paper's rule for the partition ``boundaries``
    (b[0] = 0 < ... < b[p] = n)."""
    t = _tab(table)
    Q, A = t.shape
    T = _bytes(text)
    b = np.ascontiguousarray(np.asarray(boundaries, dtype=np.uint64))
    scratch = np.empty(Q, dtype=np.uint8)
    r, s = C.c_uint64(), C.c_uint64()
    rc = lib().oracle_route_stats(Q, A, t.ctypes.data, t.itemsize, T.ctypes.data, T.size,
                                  b.ctypes.data, b.size - 1, C.byref(r), C.byref(s), scratch.ctypes.data)
    if rc != OK:
        raise ValueError(f"oracle_route_stats failed ({rc})")
    return r.value, s.value


def lookback_stats(table, text, boundaries, k: int) -> tuple[int, int]:
    """(routes, route_steps) of the k-symbol look-back rule R_i = delta*(Q, T[b_i-k, b_i)) n S(T[b_i])."""
    t = _tab(table)
    Q, A = t.shape
    T = _bytes(text)
    b = np.ascontiguousarray(np.asarray(boundaries, dtype=np.uint64))
    scratch = np.empty(2 * Q, dtype=np.uint8)
    r, s = C.c_uint64(), C.c_uint64()
    rc = lib().oracle_lookback_stats(Q, A, t.ctypes.data, t.itemsize, T.ctypes.data, T.size, b.ctypes.data,
                                     b.size - 1, k, C.byref(r), C.byref(s), scratch.ctypes.data)
    if rc != OK:
        raise ValueError(f"oracle_lookback_stats failed ({rc})")
    return r.value, s.value


def grid_boundaries(n: int, chunk_len: int) -> list[int]:
    """The grid partition used with a forced chunk length: p = max(1, n // L) chunks of
    L bytes, remainder to the last chunk (P:81-82 with reading C7)."""
    if n == 0:
        return [0]
    p = max(1, n // chunk_len)
    return [i * chunk_len for i in range(p)] + [n]
