"""B200-native PaREM hot path: chunked, speculative DFA matching (arXiv 1412.1741).

Thin Python binding over the C ABI (include/parem.h, libparem.so).  Every step of the
path runs in the library's sm_100a kernels; this module only marshals arguments.
PyTorch supplies device memory and the current CUDA stream.  There is no CPU fallback:
matching a non-CUDA tensor, or importing without the built library, raises.

    import numpy as np, torch
    from paper_1412_1741_b200 import Dfa
    dfa = Dfa(table_u16_or_u32, start=0, accept=bool_array)
    final, accepted, count = dfa.match(torch_uint8_cuda_tensor)[:3]
"""
from __future__ import annotations

import ctypes as C
from typing import NamedTuple

import numpy as np

from . import _abi
from ._abi import (BOUNDARY_AUTO, BOUNDARY_GRID, BOUNDARY_SNAP, CANDIDATES_ENUM, CANDIDATES_PAREM, KERNEL_AUTO, KERNEL_CONV, KERNEL_LANES,
                   KERNEL_TINY, PAREM_DEAD, PAREM_EINVAL, PAREM_ESYMBOL, PAREM_OK)

__all__ = ["Dfa", "MatchResult", "ParemError", "Regex", "compile_regex", "table_to_text", "table_from_text", "options", "profile", "profile_read", "PAREM_DEAD", "PAREM_OK",
           "PAREM_ESYMBOL", "PAREM_EINVAL", "lib", "SEGMAP_DTYPE", "fold_segment_maps", "exchange_and_fold", "shard_match"]


def lib():
    return _abi.load()


class ParemError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"parem status {status}: {msg}")
        self.status = status


class MatchResult(NamedTuple):
    final_state: int          # PAREM_DEAD (0xFFFFFFFF) if the walk died
    accepted: bool
    match_count: int
    status: int
    bad_offset: int
    num_chunks: int
    routes: int               # sum |R_i|   ("calculations")
    route_steps: int          # sum |R_i| * len_i
    lookups: int = 0          # converging path: lookups issued at distinct states (multiple of 1024)

    @staticmethod
    def from_struct(r: _abi.parem_result) -> "MatchResult":
        return MatchResult(r.final_state, bool(r.accepted), r.match_count, r.status, r.bad_offset, r.num_chunks,
                           r.routes, r.route_steps, int(r.lookups_k) << 10)

    @staticmethod
    def from_bytes(b: bytes) -> "MatchResult":
        return MatchResult.from_struct(_abi.parem_result.from_buffer_copy(b))


_POLICY = {"grid": BOUNDARY_GRID, "snap": BOUNDARY_SNAP, "auto": BOUNDARY_AUTO}
_CAND = {"parem": CANDIDATES_PAREM, "enum": CANDIDATES_ENUM, "lookback": _abi.CANDIDATES_LOOKBACK}
_KERNEL = {"auto": KERNEL_AUTO, "tiny": KERNEL_TINY, "lanes": KERNEL_LANES, "conv": KERNEL_CONV}


def options(chunk_len: int = 0, boundary: str = "auto", candidates: str = "parem", kernel: str = "auto",
            ws_clean: bool = False, lookback: int = 0):
    """parem_options.  ``ws_clean`` sets PAREM_FLAG_WS_CLEAN: the workspace header is known
    to be zero (torch.zeros, or a previous completed call), so no per-call reset is issued."""
    o = _abi.parem_options()
    o.chunk_len = int(chunk_len)
    o.boundary_policy = _POLICY[boundary]
    o.candidates = _CAND[candidates]
    o.kernel = _KERNEL[kernel]
    o.flags = _abi.FLAG_WS_CLEAN if ws_clean else 0
    o.lookback = int(lookback)
    return o


class Regex(NamedTuple):
    table: np.ndarray          # uint32 [num_states, alphabet_size], row-major (parem_dfa_create layout)
    start: int
    accept: np.ndarray         # bool [num_states]
    alphabet: bytes            # symbol i = alphabet[i]

    def encode(self, text: bytes) -> np.ndarray:
        """Bytes -> symbol ids (raises on a byte outside the alphabet)."""
        lut = np.full(256, 255, dtype=np.uint8)
        lut[np.frombuffer(self.alphabet, dtype=np.uint8)] = np.arange(len(self.alphabet), dtype=np.uint8)
        ids = lut[np.frombuffer(bytes(text), dtype=np.uint8)]
        if len(self.alphabet) < 256 and (ids == 255).any():
            raise ValueError("text has bytes outside the alphabet")
        return ids


def table_to_text(table, start: int, accept, alphabet: bytes) -> str:
    """parem_table_write_text: the transition-table log file (format S:184-188).
    ``table`` uint16/uint32 [Q, A] with DEAD = all-ones, ``accept`` bool [Q]."""
    L = lib()
    t = np.ascontiguousarray(table)
    Q, A = t.shape
    t32 = np.where(t == np.iinfo(t.dtype).max, np.uint32(0xFFFFFFFF), t.astype(np.uint32)).astype(np.uint32)
    t32 = np.ascontiguousarray(t32)
    bm = np.packbits(np.asarray(accept, dtype=bool), bitorder="little")
    alp = bytes(alphabet)
    if len(alp) != A:
        raise ValueError("alphabet must name every symbol column")
    need = C.c_size_t(0)
    st = L.parem_table_write_text(Q, A, t32.ctypes.data, int(start), bm.ctypes.data, alp, None, 0, C.byref(need))
    if st != PAREM_OK:
        _err(L, st)
    buf = C.create_string_buffer(need.value)
    st = L.parem_table_write_text(Q, A, t32.ctypes.data, int(start), bm.ctypes.data, alp, buf, need.value, C.byref(need))
    if st != PAREM_OK:
        _err(L, st)
    return buf.raw[: need.value].decode("latin-1")


def table_from_text(text: str | bytes) -> Regex:
    """parem_table_read_text: the inverse of table_to_text (uint32 table, PAREM_DEAD = missing)."""
    L = lib()
    raw = text.encode("latin-1") if isinstance(text, str) else bytes(text)
    info = _abi.parem_regex_info()
    st = L.parem_table_read_text(raw, len(raw), 0, None, None, C.byref(info))
    if st != PAREM_OK:
        _err(L, st)
    Q, A = info.num_states, info.alphabet_size
    tab = np.zeros((Q, A), dtype=np.uint32)
    bm = np.zeros((Q + 7) // 8, dtype=np.uint8)
    st = L.parem_table_read_text(raw, len(raw), Q, tab.ctypes.data, bm.ctypes.data, C.byref(info))
    if st != PAREM_OK:
        _err(L, st)
    acc = np.unpackbits(bm, bitorder="little")[:Q].astype(bool)
    return Regex(tab, int(info.start_state), acc, C.string_at(C.addressof(info) + _abi.parem_regex_info.alphabet.offset, A))


def compile_regex(pattern: str | bytes, alphabet: str | bytes | None = None, search: bool = False,
                  max_states: int = 1 << 16) -> Regex:
    """parem_regex_compile: the paper's RE language (Table III) -> minimal DFA (NEXT-3).
    ``search=True`` compiles Sigma* R (match count = occurrence end positions)."""
    L = lib()
    pat = pattern.encode("latin-1") if isinstance(pattern, str) else bytes(pattern)
    alp = None if alphabet is None else (alphabet.encode("latin-1") if isinstance(alphabet, str) else bytes(alphabet))
    info = _abi.parem_regex_info()
    fl = _abi.REGEX_SEARCH if search else 0
    st = L.parem_regex_compile(pat, alp, fl, 0, None, None, C.byref(info))
    if st != PAREM_OK:
        _err(L, st)
    Q, A = info.num_states, info.alphabet_size
    tab = np.zeros((Q, A), dtype=np.uint32)
    bm = np.zeros((Q + 7) // 8, dtype=np.uint8)
    st = L.parem_regex_compile(pat, alp, fl, Q, tab.ctypes.data, bm.ctypes.data, C.byref(info))
    if st != PAREM_OK:
        _err(L, st)
    acc = np.unpackbits(bm, bitorder="little")[:Q].astype(bool)
    return Regex(tab, int(info.start_state), acc, C.string_at(C.addressof(info) + _abi.parem_regex_info.alphabet.offset, A))


def profile(enable: bool = True) -> None:
    """parem_profile: record CUDA events around every kernel of later matches (this thread)."""
    lib().parem_profile(1 if enable else 0)


def profile_read() -> list[tuple[int, str, float]]:
    """(match index, kernel name, device ms) for every kernel launch recorded since
    profile(True), in launch order."""
    L = lib()
    n = C.c_int(0)
    st = L.parem_profile_read(None, 0, C.byref(n))
    if st != PAREM_OK:
        _err(L, st)
    buf = (_abi.parem_kernel_time * max(1, n.value))()
    st = L.parem_profile_read(buf, n.value, C.byref(n))
    if st != PAREM_OK:
        _err(L, st)
    return [(int(buf[i].match), buf[i].name.decode(), float(buf[i].ms)) for i in range(n.value)]


# parem_segmap_entry (include/parem.h): one per entering state of a segment
SEGMAP_DTYPE = np.dtype([("match_count", "<u8"), ("end_state", "<u4"), ("valid", "<u4")])


def fold_segment_maps(num_states: int, start: int, accept, maps, statuses, bad_offsets, seg_offsets) -> "MatchResult":
    """parem_fold_segment_maps: fold G segment maps (array (G, num_states) of SEGMAP_DTYPE)
    along q0's path -- the join of P:70 over the segments of a sharded input.  Host only."""
    L = lib()
    m = np.ascontiguousarray(maps, dtype=SEGMAP_DTYPE)
    G = m.shape[0] if m.ndim == 2 else 0
    a = np.asarray(accept)
    bm = np.packbits(a.astype(bool), bitorder="little") if a.dtype == bool else np.ascontiguousarray(a, np.uint8)
    st = np.ascontiguousarray(statuses, dtype=np.int32)
    bo = np.ascontiguousarray(bad_offsets, dtype=np.uint64)
    so = np.ascontiguousarray(seg_offsets, dtype=np.uint64)
    r = _abi.parem_result()
    rc = L.parem_fold_segment_maps(num_states, start, bm.ctypes.data, m.ctypes.data, G, st.ctypes.data, bo.ctypes.data,
                                   so.ctypes.data, C.byref(r))
    if rc not in (PAREM_OK, PAREM_ESYMBOL):
        _err(L, rc)
    return MatchResult.from_struct(r)


def exchange_and_fold(segmap, status: int, bad_offset: int, seg_offset: int, num_states: int, start: int,
                      accept_bitmap, group=None, device=None) -> "MatchResult":
    """The exchange step of a sharded match: ONE all-gather of every rank's segment map
    (num_states x 16 bytes) and (status, bad offset, segment offset), then the fold along
    q0's path on every rank.  Works on any torch.distributed backend (NCCL on GPUs, gloo
    on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    mine = torch.from_numpy(np.ascontiguousarray(segmap, dtype=SEGMAP_DTYPE).view(np.uint8).copy()).to(dev)
    meta = torch.tensor([status, bad_offset, seg_offset], dtype=torch.int64, device=dev)
    allm = torch.empty(world * mine.numel(), dtype=torch.uint8, device=dev)
    allmeta = torch.empty(world * 3, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allm, mine, group=group)
    dist.all_gather_into_tensor(allmeta, meta, group=group)
    maps = allm.cpu().numpy().view(SEGMAP_DTYPE).reshape(world, num_states)
    mt = allmeta.cpu().numpy().reshape(world, 3)
    return fold_segment_maps(num_states, start, accept_bitmap, maps, mt[:, 0], mt[:, 1].astype(np.uint64),
                             mt[:, 2].astype(np.uint64))


def shard_match(dfa: "Dfa", x_local, prev_symbol: int, seg_offset: int, group=None) -> "MatchResult":
    """One input sharded over the ranks of a torch.distributed group: this
    rank's segment map (parem_segment_map over the paper's candidate set for its first
    position), then exchange_and_fold.  ``prev_symbol`` = last byte of the previous rank's
    segment (-1 on rank 0), ``seg_offset`` = global offset of this segment's first byte."""
    import torch.distributed as dist

    m, status, bad = dfa.segment_map(x_local, prev_symbol)
    dev = x_local.device if dist.get_backend(group) == "nccl" else None
    return exchange_and_fold(m, status, bad, seg_offset, dfa.Q, dfa.start, dfa.accept_bitmap, group, dev)


def _err(L, status: int):
    raise ParemError(status, L.parem_last_error().decode(errors="replace"))


def _cuda_u8(x):
    import torch

    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("input must be a CUDA torch.Tensor (no CPU fallback)")
    if x.dtype != torch.uint8 or not x.is_contiguous():
        raise TypeError("input must be a contiguous uint8 tensor")
    return x


def _stream(stream):
    import torch

    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


class Dfa:
    """A DFA handle on the current CUDA device (parem_dfa_create).

    table  -- (Q, A) uint16/uint32 array, table[s, c] = delta(s, c); all-ones = DEAD.
    start  -- q0.
    accept -- bool[Q] (or an LSB-first bitmap of ceil(Q/8) bytes).
    """

    def __init__(self, table, start: int, accept):
        self._L = lib()
        t = np.ascontiguousarray(table)
        if t.ndim != 2 or t.dtype not in (np.uint16, np.uint32):
            raise TypeError("table must be a 2-D uint16/uint32 array")
        Q, A = t.shape
        a = np.asarray(accept)
        bm = np.packbits(a.astype(bool), bitorder="little") if a.dtype == bool else np.ascontiguousarray(a, np.uint8)
        if bm.size < (Q + 7) // 8:
            raise ValueError("accept bitmap too short")
        h = C.c_void_p()
        st = self._L.parem_dfa_create(Q, A, t.ctypes.data, t.itemsize, int(start), bm.ctypes.data, C.byref(h))
        if st != PAREM_OK:
            _err(self._L, st)
        self._h = h
        self.Q, self.A, self.start = Q, A, int(start)
        self.accept_bitmap = bm[: (Q + 7) // 8].copy()

    # -- lifetime --
    def close(self):
        if getattr(self, "_h", None):
            self._L.parem_dfa_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- introspection --
    def info(self) -> dict:
        i = _abi.parem_dfa_info()
        st = self._L.parem_dfa_get_info(self._h, C.byref(i))
        if st != PAREM_OK:
            _err(self._L, st)
        return {f: getattr(i, f) for f, _ in i._fields_}

    def plan(self, n: int, opts=None) -> dict:
        p = _abi.parem_plan_info()
        st = self._L.parem_plan(self._h, n, C.byref(opts) if opts is not None else None, C.byref(p))
        if st != PAREM_OK:
            _err(self._L, st)
        return {f: getattr(p, f) for f, _ in p._fields_ if f != "reserved"}

    def workspace_bytes(self, n: int, opts=None) -> int:
        ws = self._L.parem_workspace_bytes(self._h, n, C.byref(opts) if opts is not None else None)
        if ws == 0:
            _err(self._L, PAREM_EINVAL)
        return ws

    # -- matching --
    def match(self, x, opts=None, stream=None, **kw) -> MatchResult:
        """Synchronous match of a CUDA uint8 tensor (parem_match)."""
        x = _cuda_u8(x)
        opts = opts if opts is not None else (options(**kw) if kw else None)
        r = _abi.parem_result()
        st = self._L.parem_match(self._h, C.c_void_p(x.data_ptr()), x.numel(),
                                 C.byref(opts) if opts is not None else None, C.byref(r), _stream(stream))
        if st not in (PAREM_OK, PAREM_ESYMBOL):
            _err(self._L, st)
        return MatchResult.from_struct(r)

    def match_async(self, x, ws, result, opts=None, stream=None, n: int | None = None) -> None:
        """Enqueue parem_match_async; ``ws`` is a CUDA uint8 workspace tensor and ``result`` a
        CUDA uint8 tensor of >= 56 bytes that receives the parem_result."""
        x = _cuda_u8(x)
        n = x.numel() if n is None else n
        st = self._L.parem_match_async(self._h, C.c_void_p(x.data_ptr()), n, C.c_void_p(ws.data_ptr()), ws.numel(),
                                       C.byref(opts) if opts is not None else None, C.c_void_p(result.data_ptr()),
                                       _stream(stream))
        if st != PAREM_OK:
            _err(self._L, st)

    def batch_workspace_bytes(self, n: int, count: int, opts=None) -> int:
        ws = self._L.parem_batch_workspace_bytes(self._h, n, count, C.byref(opts) if opts is not None else None)
        if ws == 0:
            _err(self._L, PAREM_EINVAL)
        return ws

    def match_batch_async(self, x, ws, results, opts=None, stream=None) -> None:
        """Enqueue parem_match_batch_async: ``x`` is a CUDA uint8 tensor of shape (count, n)
        (count independent inputs, contiguous); ``results`` a CUDA uint8 tensor of at least
        56 * count bytes receiving one parem_result per input."""
        x = _cuda_u8(x)
        if x.dim() != 2:
            raise TypeError("batch input must be a 2-D (count, n) tensor")
        count, n = x.shape
        st = self._L.parem_match_batch_async(self._h, C.c_void_p(x.data_ptr()), n, count, C.c_void_p(ws.data_ptr()),
                                             ws.numel(), C.byref(opts) if opts is not None else None,
                                             C.c_void_p(results.data_ptr()), _stream(stream))
        if st != PAREM_OK:
            _err(self._L, st)

    def match_batch(self, x, opts=None) -> list:
        """Synchronous batched match of a (count, n) CUDA uint8 tensor: one MatchResult per row."""
        import torch

        x = _cuda_u8(x)
        count, n = x.shape
        ws = torch.zeros(self.batch_workspace_bytes(n, count, opts), dtype=torch.uint8, device=x.device)
        res = torch.zeros(max(1, count) * 56, dtype=torch.uint8, device=x.device)
        self.match_batch_async(x, ws, res, opts)
        b = res.cpu().numpy().tobytes()
        return [MatchResult.from_bytes(b[56 * i: 56 * (i + 1)]) for i in range(count)]

    def segment_map(self, x, prev_symbol: int, opts=None):
        """parem_segment_map: this segment's map over the candidate set of its first
        position (L(prev_symbol); {q0} if prev_symbol < 0).  Returns (map array of
        SEGMAP_DTYPE with num_states entries, status, local bad offset)."""
        x = _cuda_u8(x)
        m = np.zeros(self.Q, dtype=SEGMAP_DTYPE)
        st = C.c_int32(0)
        bad = C.c_uint64(0)
        rc = self._L.parem_segment_map(self._h, C.c_void_p(x.data_ptr()) if x.numel() else None, x.numel(),
                                       int(prev_symbol), C.byref(opts) if opts is not None else None, m.ctypes.data,
                                       C.byref(st), C.byref(bad), _stream(None))
        if rc != PAREM_OK:
            _err(self._L, rc)
        return m, int(st.value), int(bad.value)

    def find_workspace_bytes(self, n: int, opts=None) -> int:
        ws = self._L.parem_find_workspace_bytes(self._h, n, C.byref(opts) if opts is not None else None)
        if ws == 0:
            _err(self._L, PAREM_EINVAL)
        return ws

    def find_async(self, x, ws, positions, result, opts=None, stream=None) -> None:
        """Enqueue parem_find_async: the match plus its match END offsets (uint64, ascending)
        into the CUDA tensor ``positions`` (at most positions.numel() are written)."""
        x = _cuda_u8(x)
        st = self._L.parem_find_async(self._h, C.c_void_p(x.data_ptr()), x.numel(), C.c_void_p(ws.data_ptr()),
                                      ws.numel(), C.byref(opts) if opts is not None else None,
                                      C.c_void_p(positions.data_ptr()) if positions.numel() else None,
                                      positions.numel(), C.c_void_p(result.data_ptr()), _stream(stream))
        if st != PAREM_OK:
            _err(self._L, st)

    def find(self, x, max_positions: int | None = None, opts=None):
        """Synchronous find: (MatchResult, positions as a CUDA int64 tensor of
        min(match_count, max_positions) offsets).  max_positions=None sizes for every byte."""
        import torch

        x = _cuda_u8(x)
        cap = x.numel() if max_positions is None else int(max_positions)
        ws = torch.zeros(self.find_workspace_bytes(x.numel(), opts), dtype=torch.uint8, device=x.device)
        pos = torch.empty(max(cap, 1), dtype=torch.int64, device=x.device)
        res = torch.zeros(64, dtype=torch.uint8, device=x.device)
        self.find_async(x, ws, pos[:cap], res, opts)
        r = MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
        return r, pos[: min(cap, r.match_count)]

    def trace_async(self, x, ws, lo: int, hi: int, states, result, opts=None, stream=None) -> None:
        """Enqueue parem_trace_async: the match plus the visited states q_{k+1}, lo <= k < hi,
        into the CUDA int32/uint32 tensor ``states`` (hi - lo entries)."""
        x = _cuda_u8(x)
        if states.numel() < hi - lo:
            raise ValueError("states tensor smaller than the window")
        st = self._L.parem_trace_async(self._h, C.c_void_p(x.data_ptr()), x.numel(), C.c_void_p(ws.data_ptr()),
                                       ws.numel(), C.byref(opts) if opts is not None else None, int(lo), int(hi),
                                       C.c_void_p(states.data_ptr()) if hi > lo else None,
                                       C.c_void_p(result.data_ptr()), _stream(stream))
        if st != PAREM_OK:
            _err(self._L, st)

    def trace(self, x, lo: int = 0, hi: int | None = None, opts=None):
        """Synchronous route trace (Alg. 1's Rr of the selected routes): (MatchResult, CUDA int64
        tensor of the states after symbols lo .. hi-1; PAREM_DEAD = 0xFFFFFFFF after death)."""
        import torch

        x = _cuda_u8(x)
        hi = x.numel() if hi is None else int(hi)
        ws = torch.zeros(self.find_workspace_bytes(x.numel(), opts), dtype=torch.uint8, device=x.device)
        st = torch.empty(max(hi - lo, 1), dtype=torch.int32, device=x.device)
        res = torch.zeros(64, dtype=torch.uint8, device=x.device)
        self.trace_async(x, ws, lo, hi, st, res, opts)
        r = MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
        return r, (st[: max(hi - lo, 0)].to(torch.int64) & 0xFFFFFFFF)

    def match_continue_async(self, x, offset_base: int, ws, carry, result, opts=None, stream=None) -> None:
        x = _cuda_u8(x)
        st = self._L.parem_match_continue_async(
            self._h, C.c_void_p(x.data_ptr()), x.numel(), offset_base, C.c_void_p(ws.data_ptr()), ws.numel(),
            C.byref(opts) if opts is not None else None, C.c_void_p(carry.data_ptr()) if carry is not None else None,
            C.c_void_p(result.data_ptr()), _stream(stream))
        if st != PAREM_OK:
            _err(self._L, st)

    def match_host(self, x, opts=None, stream=None) -> MatchResult:
        """End-to-end match of a HOST buffer (numpy uint8 array or CPU torch tensor; pinned
        memory recommended): parem_match_host pipelines H2D copies with matching."""
        try:
            import torch

            if isinstance(x, torch.Tensor):
                if x.is_cuda or x.dtype != torch.uint8 or not x.is_contiguous():
                    raise TypeError("host input must be a contiguous CPU uint8 tensor")
                ptr, n = x.data_ptr(), x.numel()
            else:
                raise ImportError
        except ImportError:
            a = np.ascontiguousarray(x, dtype=np.uint8)
            ptr, n = a.ctypes.data, a.size
        r = _abi.parem_result()
        st = self._L.parem_match_host(self._h, C.c_void_p(ptr), n, C.byref(opts) if opts is not None else None,
                                      C.byref(r), _stream(stream))
        if st not in (PAREM_OK, PAREM_ESYMBOL):
            _err(self._L, st)
        return MatchResult.from_struct(r)
