"""ctypes declarations of the C ABI in include/parem.h (argument marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("PAREM_LIB") or os.path.join(_HERE, "libparem.so")

PAREM_OK, PAREM_EINVAL, PAREM_ESYMBOL, PAREM_ECUDA, PAREM_ENOMEM, PAREM_EINTERNAL = 0, -1, -2, -3, -4, -5
PAREM_DEAD = 0xFFFFFFFF
BOUNDARY_GRID, BOUNDARY_SNAP, BOUNDARY_AUTO = 0, 1, 2
CANDIDATES_PAREM, CANDIDATES_ENUM, CANDIDATES_LOOKBACK = 0, 1, 2
KERNEL_AUTO, KERNEL_TINY, KERNEL_LANES, KERNEL_CONV = 0, 1, 2, 3


class parem_result(C.Structure):
    _fields_ = [("match_count", C.c_uint64), ("final_state", C.c_uint32), ("accepted", C.c_uint32),
                ("bad_offset", C.c_uint64), ("num_chunks", C.c_uint64), ("routes", C.c_uint64),
                ("route_steps", C.c_uint64), ("status", C.c_int32), ("lookups_k", C.c_uint32)]


class parem_options(C.Structure):
    _fields_ = [("chunk_len", C.c_uint64), ("boundary_policy", C.c_uint32), ("candidates", C.c_uint32),
                ("kernel", C.c_uint32), ("flags", C.c_uint32), ("lookback", C.c_uint32), ("reserved", C.c_uint32)]


FLAG_WS_CLEAN = 1


class parem_kernel_time(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("ms", C.c_float), ("match", C.c_uint32)]


REGEX_SEARCH = 1


class parem_regex_info(C.Structure):
    _fields_ = [("num_states", C.c_uint32), ("alphabet_size", C.c_uint32), ("start_state", C.c_uint32),
                ("reserved", C.c_uint32), ("alphabet", C.c_char * 256)]


class parem_dfa_info(C.Structure):
    _fields_ = [("num_states", C.c_uint32), ("internal_states", C.c_uint32), ("alphabet_size", C.c_uint32),
                ("has_sink", C.c_uint32), ("min_L", C.c_uint32), ("max_L", C.c_uint32), ("sum_L", C.c_uint64),
                ("start_state", C.c_uint32), ("table_class", C.c_uint32), ("device_bytes", C.c_uint64)]


class parem_plan_info(C.Structure):
    _fields_ = [("kernel", C.c_uint32), ("block_threads", C.c_uint32), ("grid_blocks", C.c_uint64),
                ("num_chunks", C.c_uint64), ("chunk_len", C.c_uint64), ("boundary_policy", C.c_uint32),
                ("candidates", C.c_uint32), ("slots", C.c_uint32), ("symbols_per_lookup", C.c_uint32),
                ("smem_bytes", C.c_size_t), ("workspace_bytes", C.c_size_t), ("snap_window", C.c_uint32),
                ("reserved", C.c_uint32)]


assert C.sizeof(parem_result) == 56
assert C.sizeof(parem_options) == 32

EXPORTS = [
    "parem_dfa_create", "parem_dfa_destroy", "parem_workspace_bytes", "parem_match_async",
    "parem_match_continue_async", "parem_match", "parem_match_host", "parem_dfa_get_info", "parem_plan",
    "parem_last_error", "parem_version", "parem_bench_read_stream", "parem_bench_gather", "parem_profile",
    "parem_profile_read", "parem_regex_compile", "parem_table_write_text", "parem_table_read_text", "parem_find_async", "parem_find_workspace_bytes", "parem_trace_async",
    "parem_batch_workspace_bytes", "parem_match_batch_async", "parem_segment_map", "parem_fold_segment_maps",
]

_LIB = None


def load(path: str = SO_PATH):
    """Load libparem.so and declare every exported signature.  Raises if the CUDA library
    is missing -- there is no CPU fallback."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built -- run `python buildlib.py` (no CPU fallback exists)")
    L = C.CDLL(path)
    u32, u64, vp, i32, sz = C.c_uint32, C.c_uint64, C.c_void_p, C.c_int, C.c_size_t
    R, O = C.POINTER(parem_result), C.POINTER(parem_options)
    L.parem_dfa_create.restype = i32
    L.parem_dfa_create.argtypes = [u32, u32, vp, u32, u32, vp, C.POINTER(vp)]
    L.parem_dfa_destroy.restype = i32
    L.parem_dfa_destroy.argtypes = [vp]
    L.parem_workspace_bytes.restype = sz
    L.parem_workspace_bytes.argtypes = [vp, u64, O]
    L.parem_match_async.restype = i32
    L.parem_match_async.argtypes = [vp, vp, u64, vp, sz, O, vp, vp]
    L.parem_match_continue_async.restype = i32
    L.parem_match_continue_async.argtypes = [vp, vp, u64, u64, vp, sz, O, vp, vp, vp]
    L.parem_batch_workspace_bytes.restype = sz
    L.parem_batch_workspace_bytes.argtypes = [vp, u64, u64, O]
    L.parem_match_batch_async.restype = i32
    L.parem_match_batch_async.argtypes = [vp, vp, u64, u64, vp, sz, O, vp, vp]
    L.parem_segment_map.restype = i32
    L.parem_segment_map.argtypes = [vp, vp, u64, C.c_int32, O, vp, C.POINTER(C.c_int32), C.POINTER(u64), vp]
    L.parem_fold_segment_maps.restype = i32
    L.parem_fold_segment_maps.argtypes = [u32, u32, vp, vp, u32, vp, vp, vp, R]
    L.parem_match.restype = i32
    L.parem_match.argtypes = [vp, vp, u64, O, R, vp]
    L.parem_match_host.restype = i32
    L.parem_match_host.argtypes = [vp, vp, u64, O, R, vp]
    L.parem_find_workspace_bytes.restype = sz
    L.parem_find_workspace_bytes.argtypes = [vp, u64, O]
    L.parem_find_async.restype = i32
    L.parem_find_async.argtypes = [vp, vp, u64, vp, sz, O, vp, u64, vp, vp]
    L.parem_trace_async.restype = i32
    L.parem_trace_async.argtypes = [vp, vp, u64, vp, sz, O, u64, u64, vp, vp, vp]
    L.parem_regex_compile.restype = i32
    L.parem_regex_compile.argtypes = [C.c_char_p, C.c_char_p, u32, u32, vp, vp, C.POINTER(parem_regex_info)]
    L.parem_table_write_text.restype = i32
    L.parem_table_write_text.argtypes = [u32, u32, vp, u32, vp, C.c_char_p, vp, sz, C.POINTER(sz)]
    L.parem_table_read_text.restype = i32
    L.parem_table_read_text.argtypes = [C.c_char_p, sz, u32, vp, vp, C.POINTER(parem_regex_info)]
    L.parem_profile.restype = i32
    L.parem_profile.argtypes = [i32]
    L.parem_profile_read.restype = i32
    L.parem_profile_read.argtypes = [C.POINTER(parem_kernel_time), i32, C.POINTER(i32)]
    L.parem_dfa_get_info.restype = i32
    L.parem_dfa_get_info.argtypes = [vp, C.POINTER(parem_dfa_info)]
    L.parem_plan.restype = i32
    L.parem_plan.argtypes = [vp, u64, O, C.POINTER(parem_plan_info)]
    L.parem_last_error.restype = C.c_char_p
    L.parem_last_error.argtypes = []
    L.parem_version.restype = C.c_char_p
    L.parem_version.argtypes = []
    L.parem_bench_read_stream.restype = C.c_float
    L.parem_bench_read_stream.argtypes = [vp, u64, vp, i32, vp]
    L.parem_bench_gather.restype = C.c_float
    L.parem_bench_gather.argtypes = [u32, vp, u32, u32, vp, C.POINTER(u64), i32, vp]
    _LIB = L
    return L
