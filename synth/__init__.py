"""Seeded synthetic inputs -- shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: it only produces byte strings and DFA tables
(row-major ``table[s*A + c]``, uint16/uint32, DEAD = all-ones of the element width).
The five BASELINE.json configurations are described by :func:`config`.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(so):
            import buildlib  # noqa: WPS433  (repo root on sys.path)

            buildlib.build_synth()
        L = C.CDLL(so)
        u64, u32, p = C.c_uint64, C.c_uint32, C.c_void_p
        L.synth_draw.restype = u64
        L.synth_draw.argtypes = [u64, u64, u64]
        L.synth_below.restype = u32
        L.synth_below.argtypes = [u64, u64, u64, u32]
        L.synth_bernoulli_threshold.restype = u64
        L.synth_bernoulli_threshold.argtypes = [C.c_double]
        L.synth_uniform_symbols.argtypes = [p, u64, u32, u64, u64, u64]
        L.synth_bernoulli.argtypes = [p, u64, C.c_double, u64, u64]
        L.synth_random_dfa.argtypes = [p, u32, u32, u32, u64]
        L.synth_sparse_dfa.argtypes = [p, u32, u32, u32, u32, u64]
        L.synth_partial_dfa.argtypes = [p, u32, u32, u32, C.c_double, u64]
        L.synth_kmp_dfa.restype = C.c_int
        L.synth_kmp_dfa.argtypes = [p, u32, p, u32, u32]
        L.synth_markov_bytes.argtypes = [p, u64, u64]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def draw(seed: int, stream: int, index: int) -> int:
    return lib().synth_draw(seed, stream, index)


def uniform_symbols(n: int, A: int, seed: int, stream: int = 0, offset: int = 0, out=None) -> np.ndarray:
    out = np.empty(n, dtype=np.uint8) if out is None else out
    assert out.dtype == np.uint8 and out.flags.c_contiguous and out.size >= n
    if n:
        lib().synth_uniform_symbols(_ptr(out), n, A, seed, stream, offset)
    return out


def bernoulli(n: int, p: float, seed: int, stream: int = 2) -> np.ndarray:
    out = np.empty(n, dtype=np.uint8)
    if n:
        lib().synth_bernoulli(_ptr(out), n, p, seed, stream)
    return out.astype(bool)


def random_dfa(Q: int, A: int, seed: int, dtype=np.uint16) -> np.ndarray:
    t = np.empty(Q * A, dtype=dtype)
    lib().synth_random_dfa(_ptr(t), t.itemsize, Q, A, seed)
    return t.reshape(Q, A)


def sparse_dfa(Q: int, A: int, targets: int, seed: int, dtype=np.uint16) -> np.ndarray:
    t = np.empty(Q * A, dtype=dtype)
    lib().synth_sparse_dfa(_ptr(t), t.itemsize, Q, A, targets, seed)
    return t.reshape(Q, A)


def partial_dfa(Q: int, A: int, p_dead: float, seed: int, dtype=np.uint16) -> np.ndarray:
    t = np.empty(Q * A, dtype=dtype)
    lib().synth_partial_dfa(_ptr(t), t.itemsize, Q, A, p_dead, seed)
    return t.reshape(Q, A)


def kmp_dfa(pattern, A: int, dtype=np.uint16) -> np.ndarray:
    """Sigma*P search automaton, states 0..m, accept {m}."""
    P = np.ascontiguousarray(np.asarray(pattern, dtype=np.uint8))
    m = int(P.size)
    t = np.empty((m + 1) * A, dtype=dtype)
    rc = lib().synth_kmp_dfa(_ptr(t), t.itemsize, _ptr(P), m, A)
    if rc != 0:
        raise ValueError("bad pattern")
    return t.reshape(m + 1, A)


def markov_bytes(n: int, seed: int, out=None) -> np.ndarray:
    out = np.empty(n, dtype=np.uint8) if out is None else out
    if n:
        lib().synth_markov_bytes(_ptr(out), n, seed)
    return out


def pack_bitmap(flags) -> np.ndarray:
    """LSB-first accept bitmap (the ABI's format), ceil(Q/8) bytes."""
    f = np.asarray(flags, dtype=bool)
    return np.packbits(f, bitorder="little")


# --------------------------------------------------------------------------------------
# The five BASELINE.json configurations (recipes in SURVEY.md §8(d), fixed in DESIGN.md)
# --------------------------------------------------------------------------------------

@dataclass
class Config:
    index: int
    name: str
    table: np.ndarray          # (Q, A) uint16/uint32
    start: int
    accept: np.ndarray         # bool[Q]
    n: int
    input_kind: str            # "uniform" | "markov"
    input_seed: int
    meta: dict = field(default_factory=dict)

    @property
    def Q(self) -> int:
        return int(self.table.shape[0])

    @property
    def A(self) -> int:
        return int(self.table.shape[1])

    def make_input(self, n: int | None = None, out=None) -> np.ndarray:
        n = self.n if n is None else n
        if self.input_kind == "markov":
            return markov_bytes(n, self.input_seed, out=out)
        return uniform_symbols(n, self.A, self.input_seed, 0, 0, out=out)


def cfg2_pattern() -> np.ndarray:
    return uniform_symbols(12, 4, seed=2, stream=3)


def config(k: int, n: int | None = None) -> Config:
    """BASELINE.json configs[k-1] (k = 1..5).  ``n`` overrides the input length
    (the CI-sized variants use n = 2^20)."""
    if k == 1:
        # (a|b)*abb, KMP numbering (reading C14): rows 0..3, columns a=0, b=1
        t = np.array([[1, 0], [1, 2], [1, 3], [1, 0]], dtype=np.uint32)
        acc = np.array([False, False, False, True])
        c = Config(1, "cfg1 (a|b)*abb, 4 states, u32, 1 MiB", t, 0, acc, 1 << 20, "uniform", 0)
    elif k == 2:
        P = cfg2_pattern()
        t = kmp_dfa(P, 4, np.uint16)
        acc = np.zeros(13, dtype=bool)
        acc[12] = True
        c = Config(2, "cfg2 DNA 12-mer KMP, 13 states, 1 GiB", t, 0, acc, 1 << 30, "uniform", 2,
                   {"pattern": P.tolist()})
    elif k == 3:
        t = random_dfa(256, 26, seed=1, dtype=np.uint16)
        acc = bernoulli(256, 0.1, seed=1, stream=2)
        c = Config(3, "cfg3 random dense 256x26, 4 GiB", t, 0, acc, 1 << 32, "uniform", 3)
    elif k == 4:
        t = sparse_dfa(4096, 256, 4, seed=4, dtype=np.uint16)
        acc = bernoulli(4096, 0.05, seed=4, stream=2)
        c = Config(4, "cfg4 sparse 4096x256 (<=4 targets/state), 2 GiB", t, 0, acc, 1 << 31, "uniform", 4)
    elif k == 5:
        t = random_dfa(1024, 256, seed=5, dtype=np.uint16)
        acc = bernoulli(1024, 0.1, seed=5, stream=2)
        c = Config(5, "cfg5 dense 1024x256, order-1 Markov input, 4 GiB", t, 0, acc, 1 << 32, "markov", 5)
    else:
        raise ValueError(k)
    if n is not None:
        c.n = n
    return c
