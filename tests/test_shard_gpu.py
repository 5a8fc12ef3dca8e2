"""SURVEY §8(e) on one GPU: an input split into G segments, each segment's map computed on
the device (parem_segment_map: the paper's candidate set for the segment's first position,
R = L(previous byte)), folded along q0's path (parem_fold_segment_maps) -- equal to
the oracle's walk of the whole input; the maps themselves equal the oracle's walk of the
segment from every candidate."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod(cuda_device):
    import torch

    return torch


@pytest.fixture(scope="module")
def parem(cuda_device):
    import paper_1412_1741_b200 as P

    P.lib()
    return P


def sharded(parem, torch, table, start, acc, x, cuts):
    maps, st, bad = [], [], []
    with parem.Dfa(table, start, acc) as d:
        for g in range(len(cuts) - 1):
            seg = torch.from_numpy(np.ascontiguousarray(x[cuts[g]:cuts[g + 1]])).cuda()
            prev = int(x[cuts[g] - 1]) if g > 0 else -1
            m, s, b = d.segment_map(seg, prev)
            maps.append(m)
            st.append(s)
            bad.append(b)
        bm = d.accept_bitmap
    return parem.fold_segment_maps(table.shape[0], start, bm, np.stack(maps), st, bad, cuts[:-1]), maps


def expect(parem, torch, table, start, acc, x, cuts):
    got, maps = sharded(parem, torch, table, start, acc, x, cuts)
    ref = oracle.walk(table, start, acc, x)
    if ref.status == oracle.ESYMBOL:
        assert (got.status, got.bad_offset) == (ref.status, ref.bad_offset)
    else:
        assert (got.final_state, got.accepted, got.match_count, got.status) == \
            (ref.final_state, ref.accepted, ref.match_count, 0), (got, ref)
    return maps


@pytest.mark.parametrize("k", [1, 2, 3, 5])
@pytest.mark.parametrize("G", [2, 3, 5])
def test_sharded_configs(parem, torch_mod, k, G):
    c = synth.config(k, n=(3 << 20) + 333)
    x = c.make_input()
    cuts = [int(v) for v in np.linspace(0, x.size, G + 1)]
    cuts[1] += 5                                   # uneven
    expect(parem, torch_mod, c.table, c.start, c.accept, x, cuts)


def test_segment_map_entries_equal_oracle(parem, torch_mod):
    c = synth.config(3, n=1 << 20)
    x = c.make_input()
    cuts = [0, 300_001, x.size]
    maps = expect(parem, torch_mod, c.table, c.start, c.accept, x, cuts)
    seg, prev = x[cuts[1]:], int(x[cuts[1] - 1])
    R = sorted({int(v) for v in c.table[:, prev]})
    m = maps[1]
    assert [int(i) for i in np.nonzero(m["valid"])[0]] == R
    for r in R[::7]:
        w = oracle.walk(c.table, r, c.accept, seg)
        assert (int(m[r]["end_state"]), int(m[r]["match_count"])) == (w.final_state, w.match_count), r


def test_sharded_partial_and_non_merging(parem, torch_mod):
    t = synth.partial_dfa(40, 5, 0.05, 11)          # DEAD entries: lanes kernel, sink
    acc = synth.bernoulli(40, 0.2, 11)
    x = synth.uniform_symbols(200_000, 5, 12)
    expect(parem, torch_mod, t, 0, acc, x, [0, 70_000, 140_001, x.size])
    Q, A = 7, 4                                      # permutation columns: routes never merge
    tp = np.array([[(q + c + 1) % Q for c in range(A)] for q in range(Q)], dtype=np.uint16)
    accp = np.zeros(Q, dtype=bool)
    accp[3] = True
    xp = synth.uniform_symbols(100_000, A, 13)
    expect(parem, torch_mod, tp, 0, accp, xp, [0, 50_000, xp.size])


def test_sharded_esymbol_and_empty(parem, torch_mod):
    c = synth.config(2, n=300_000)
    x = c.make_input().copy()
    x[200_123] = 7
    expect(parem, torch_mod, c.table, c.start, c.accept, x, [0, 100_000, 200_000, x.size])
    y = c.make_input()
    expect(parem, torch_mod, c.table, c.start, c.accept, y, [0, 150_000, 150_000, y.size])   # empty middle


def test_sharded_empty_candidate_set_still_validates(parem, torch_mod):
    """R = L(previous byte) can be empty (C10: only the sink arrives); the segment's bytes
    are still validated (C11) -- found by tools/stress.py (seed 537)."""
    D = 0xFFFF
    t = np.array([[1, D, 0], [D, D, D]], dtype=np.uint16)   # L(symbol 1) = {} : every entry DEAD
    acc = np.array([False, True])
    x = np.array([0, 1, 2, 9, 0, 2], dtype=np.uint8)         # invalid 9 at offset 3
    expect(parem, torch_mod, t, 0, acc, x, [0, 2, x.size])
    y = np.array([0, 1, 2, 0, 0, 2], dtype=np.uint8)         # valid: the walk died at offset 1
    expect(parem, torch_mod, t, 0, acc, y, [0, 2, 4, y.size])
