"""CPU-side checks of the C ABI: the library loads, exports every symbol include/parem.h
declares, and rejects bad arguments before touching the device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import buildlib

    buildlib.build_parem()
    from paper_1412_1741_b200 import _abi

    return _abi.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "parem.h")).read()
    return sorted(set(re.findall(r"\b(parem_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    from paper_1412_1741_b200 import _abi

    assert set(_abi.EXPORTS) == set(names)


def test_version_and_error_string(L):
    assert b"sm_100a" in L.parem_version()
    assert isinstance(L.parem_last_error(), bytes)


def _create(L, t, start=0, acc=None):
    t = np.ascontiguousarray(t)
    Q = t.shape[0] if t.ndim == 2 else 0
    A = t.shape[1] if t.ndim == 2 else 0
    bm = np.packbits(np.zeros(max(Q, 1), dtype=bool) if acc is None else acc, bitorder="little")
    h = C.c_void_p()
    return L.parem_dfa_create(Q, A, t.ctypes.data, t.itemsize, start, bm.ctypes.data, C.byref(h)), h


@pytest.mark.parametrize("table,start,why", [
    (np.zeros((0, 2), np.uint16), 0, "Q = 0"),
    (np.zeros((2, 0), np.uint16), 0, "A = 0"),
    (np.zeros((2, 257), np.uint16), 0, "A > 256"),
    (np.array([[0, 2]], np.uint16), 0, "entry >= Q and not DEAD"),
    (np.array([[0, 0]], np.uint16), 1, "start >= Q"),
    (np.zeros((3, 2), np.uint8), 0, "elem_bytes 1"),
])
def test_create_rejects_bad_arguments(L, table, start, why):
    rc, h = _create(L, table, start)
    assert rc == -1, why
    assert not h.value
    assert L.parem_last_error()


def test_create_rejects_too_many_states(L):
    # u32 device offsets: Q > 2^22 is refused before the table is read
    t = np.zeros(4, np.uint32)
    bm = np.zeros(1, np.uint8)
    h = C.c_void_p()
    rc = L.parem_dfa_create((1 << 22) + 1, 1, t.ctypes.data, 4, 0, bm.ctypes.data, C.byref(h))
    assert rc == -1 and not h.value
    assert b"4194304" in L.parem_last_error()


def test_null_handles(L):
    assert L.parem_dfa_destroy(None) == 0
    assert L.parem_workspace_bytes(None, 10, None) == 0
    from paper_1412_1741_b200 import _abi

    r = _abi.parem_result()
    assert L.parem_match(None, None, 0, None, C.byref(r), None) == -1


def test_product_path_has_no_cpu_fallback():
    """The binding refuses CPU tensors; the package never imports the oracle."""
    import ast

    pkg = os.path.join(ROOT, "paper_1412_1741_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, (ast.Import, ast.ImportFrom)):
                    mods = [a.name for a in node.names] + ([node.module] if isinstance(node, ast.ImportFrom) and node.module else [])
                    assert not any(m and m.split(".")[0] in ("oracle", "synth") for m in mods), fn
    csrc = os.path.join(pkg, "csrc")
    for fn in os.listdir(csrc):
        assert "oracle" not in open(os.path.join(csrc, fn)).read().lower(), fn
