"""Pins for the sequential oracle (oracle.c) -- each checks it against something other
than itself: textbook hand results, Python's regex engine, naive substring counting,
the one-hot x 0/1-matrix view of FA evaluation (Maine), and the paper's values."""
import itertools
import re

import numpy as np
import pytest

import oracle
import synth

AB_ABB = np.array([[1, 0], [1, 2], [1, 3], [1, 0]], dtype=np.uint32)   # reading C14
AB_ACC = np.array([False, False, False, True])


def ab(s: str):
    return [{"a": 0, "b": 1}[ch] for ch in s]


@pytest.mark.parametrize("text,final,acc,count", [
    ("abb", 3, True, 1), ("aabb", 3, True, 1), ("babb", 3, True, 1), ("abbabb", 3, True, 2),
    ("abab", 2, False, 0), ("", 0, False, 0), ("bbbb", 0, False, 0), ("abba", 1, False, 1),
])
def test_ab_abb_hand_strings(text, final, acc, count):
    """(a|b)*abb on hand-written strings (SURVEY §8(c) pins, textbook DFA)."""
    r = oracle.walk(AB_ABB, 0, AB_ACC, ab(text))
    assert (r.final_state, r.accepted, r.match_count, r.status) == (final, acc, count, 0)


def test_ab_abb_exhaustive_vs_regex():
    """All strings of length <= 12 over {a,b}: count = #prefixes fully matching (a|b)*abb
    (Python's regex engine), accept = fullmatch of the whole string."""
    pat = re.compile(r"(a|b)*abb")
    for L in range(0, 13):
        for tup in itertools.product("ab", repeat=L):
            s = "".join(tup)
            r = oracle.walk(AB_ABB, 0, AB_ACC, ab(s))
            want = sum(1 for k in range(1, L + 1) if pat.fullmatch(s[:k]))
            assert r.match_count == want, s
            assert r.accepted == bool(pat.fullmatch(s)), s


def naive_count(text: bytes, pat: bytes) -> int:
    cnt, i = 0, text.find(pat)
    while i >= 0:
        cnt += 1
        i = text.find(pat, i + 1)
    return cnt


@pytest.mark.parametrize("seed", range(8))
def test_kmp_count_vs_naive_substring(seed):
    """Sigma*P search DFA: count of accepting positions = overlapping occurrences."""
    rng = np.random.default_rng(seed)
    A = int(rng.integers(1, 6))
    m = int(rng.integers(1, 7))
    P = rng.integers(0, A, m).astype(np.uint8)
    T = rng.integers(0, A, 3000).astype(np.uint8)
    for pos in rng.integers(0, 3000 - m, 20):      # plant occurrences
        T[pos:pos + m] = P
    t = synth.kmp_dfa(P, A, np.uint32)
    acc = np.zeros(m + 1, dtype=bool)
    acc[m] = True
    r = oracle.walk(t, 0, acc, T)
    assert r.match_count == naive_count(T.tobytes(), P.tobytes())
    assert r.accepted == (T[-m:].tobytes() == P.tobytes())


def onehot_matrix_walk(table, start, accept, text):
    """FA evaluation as matrix multiplication (Maine): v_{k} = v_{k-1} M_{T[k]},
    M_c[q, q'] = 1 iff delta(q, c) = q'.  A DEAD entry is an all-zero row."""
    Q, A = table.shape
    dead = np.iinfo(table.dtype).max
    M = np.zeros((A, Q, Q), dtype=np.int64)
    for q in range(Q):
        for c in range(A):
            if table[q, c] != dead:
                M[c, q, table[q, c]] = 1
    f = np.asarray(accept, dtype=np.int64)
    v = np.zeros(Q, dtype=np.int64)
    v[start] = 1
    count = 0
    for c in text:
        v = v @ M[c]
        count += int(v @ f)
    if v.sum() == 0:
        return oracle.DEAD, False, count
    s = int(np.argmax(v))
    return s, bool(f[s]), count


@pytest.mark.parametrize("seed", range(12))
def test_random_dfa_vs_matrix_product(seed):
    rng = np.random.default_rng(100 + seed)
    Q = int(rng.choice([1, 2, 3, 5, 13, 40]))
    A = int(rng.choice([1, 2, 4, 26]))
    dt = np.uint16 if seed % 2 else np.uint32
    if seed % 3 == 0:
        t = synth.partial_dfa(Q, A, 0.08, seed, dt)
    else:
        t = synth.random_dfa(Q, A, seed, dt)
    acc = rng.random(Q) < 0.3
    q0 = int(rng.integers(0, Q))
    T = rng.integers(0, A, int(rng.integers(0, 400))).astype(np.uint8)
    r = oracle.walk(t, q0, acc, T)
    assert (r.final_state, r.accepted, r.match_count) == onehot_matrix_walk(t, q0, acc, T)


def test_parallel_worked_example():
    """The paper's worked input over Table I: one "parallel" at offsets 5..12,
    final state 0 (Table II, last route ends in 0), rejected."""
    t = synth.kmp_dfa([0, 1, 2, 1, 4, 4, 3, 4], 5, np.uint32)       # p a r e l -> 0..4
    acc = np.zeros(9, dtype=bool)
    acc[8] = True
    T = ["parel".index(ch) for ch in "plaraparallelapareparapl"]
    r = oracle.walk(t, 0, acc, T)
    assert (r.final_state, r.accepted, r.match_count) == (0, False, 1)
    r = oracle.walk(t, 0, acc, ["parel".index(ch) for ch in "parallel"])
    assert (r.final_state, r.accepted, r.match_count) == (8, True, 1)


def test_empty_input_and_start_not_counted():
    """C12: n = 0 gives (q0, q0 in F, 0).  C3: the empty prefix is not counted even when
    q0 in F; each later visit to F counts."""
    t = np.array([[0]], dtype=np.uint16)
    r = oracle.walk(t, 0, np.array([True]), [])
    assert (r.final_state, r.accepted, r.match_count) == (0, True, 0)
    r = oracle.walk(t, 0, np.array([True]), [0, 0, 0])
    assert (r.final_state, r.accepted, r.match_count) == (0, True, 3)


def test_symbol_error_smallest_offset():
    """C11: a byte >= A is ESYMBOL at the smallest offending offset, checked before the
    walk and regardless of death."""
    t = np.array([[0xFFFF, 0], [0, 0]], dtype=np.uint16)
    r = oracle.walk(t, 0, np.array([False, True]), [0, 1, 1, 7, 2, 9])
    assert r.status == oracle.ESYMBOL and r.bad_offset == 3
    r = oracle.walk(t, 0, np.array([False, True]), [1, 0, 0])
    assert r.status == 0


def test_dead_counterexample_C9():
    """C9: delta(0,a)=1, delta(0,b)=0, delta(1,a)=DEAD, delta(1,b)=0 on "aa": the walk dies
    on the second symbol with 1 hit (state 1 accepting)."""
    t = np.array([[1, 0], [0xFFFF, 0]], dtype=np.uint16)
    acc = np.array([False, True])
    r = oracle.walk(t, 0, acc, [0, 0])
    assert (r.final_state, r.accepted, r.match_count) == (oracle.DEAD, False, 1)
    r = oracle.walk(t, 0, acc, [0, 0, 1, 0])     # stays dead
    assert (r.final_state, r.accepted, r.match_count) == (oracle.DEAD, False, 1)


def test_states_at_matches_prefix_walks():
    rng = np.random.default_rng(7)
    t = synth.random_dfa(9, 3, 7, np.uint16)
    T = rng.integers(0, 3, 500).astype(np.uint8)
    offs = np.sort(rng.integers(0, 501, 30))
    st = oracle.states_at(t, 2, T, offs)
    acc = np.zeros(9, dtype=bool)
    for o, s in zip(offs, st):
        want = oracle.walk(t, 2, acc, T[:o]).final_state
        assert s == want


def test_invalid_arguments():
    t = np.array([[0, 5]], dtype=np.uint16)     # entry 5 >= Q and not DEAD
    r = oracle.walk(t, 0, np.array([False]), [1])
    assert r.status == oracle.EINVAL
    r = oracle.walk(np.array([[0]], dtype=np.uint16), 3, np.array([False]), [0])
    assert r.status == oracle.EINVAL


# ---------------------------------------------------------------- NEXT-4: match positions
def test_positions_kmp_against_substring_search():
    """Match end offsets of the Sigma*P automaton = j + |P| - 1 for every (overlapping)
    occurrence P = T[j : j + |P|], found by naive substring search."""
    rng = np.random.default_rng(11)
    for P in ([0, 1, 2, 1, 4, 4, 3, 4], [0, 0, 1], [2, 2, 2]):
        t = synth.kmp_dfa(P, 5, np.uint16)
        acc = np.zeros(len(P) + 1, dtype=bool)
        acc[-1] = True
        x = rng.integers(0, 5, 20000).astype(np.uint8)
        for pos in rng.integers(0, 20000 - len(P), 40):
            x[pos:pos + len(P)] = P
        want = [j + len(P) - 1 for j in range(x.size - len(P) + 1) if list(x[j:j + len(P)]) == list(P)]
        got, cnt = oracle.positions(t, 0, acc, x)
        assert got.tolist() == want and cnt == len(want) == oracle.walk(t, 0, acc, x).match_count


def test_positions_abb_regex_and_caps():
    """(a|b)*abb: offsets k with re.fullmatch on the prefix T[:k+1]; a cap keeps the first
    offsets and still reports the full count; DEAD stops the list (C9)."""
    t = np.array([[1, 0], [1, 2], [1, 3], [1, 0]], dtype=np.uint32)
    acc = np.array([False, False, False, True])
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2, 3000).astype(np.uint8)
    s = "".join("ab"[c] for c in x)
    want = [k for k in range(len(s)) if re.fullmatch("(a|b)*abb", s[: k + 1])]
    got, cnt = oracle.positions(t, 0, acc, x)
    assert got.tolist() == want and cnt == len(want)
    got5, cnt5 = oracle.positions(t, 0, acc, x, cap=5)
    assert got5.tolist() == want[:5] and cnt5 == len(want)
    tp = np.array([[1, 0], [0xFFFF, 3], [1, 3], [3, 3]], dtype=np.uint16)
    accp = np.array([False, True, False, True])
    got, cnt = oracle.positions(tp, 0, accp, np.array([0, 1, 0, 0, 1], np.uint8))   # 0 -a-> 1 -b-> 3 -> 3 -> 3
    assert got.tolist() == [0, 1, 2, 3, 4] and cnt == 5
    got, cnt = oracle.positions(tp, 0, accp, np.array([0, 0, 1], np.uint8))   # dies at offset 1
    assert got.tolist() == [0] and cnt == 1


# ---------------------------------------------------------------- NEXT-2 (i): k-symbol look-back
def test_lookback_k1_is_the_papers_rule():
    """k = 1: delta*(Q, T[b-1]) n S(T[b]) = L(c_last) n S(c_first), the paper's R;
    checked against the independent oracle_route_stats on complete and partial tables."""
    rng = np.random.default_rng(21)
    for seed in range(8):
        Q, A = int(rng.choice([3, 9, 40])), int(rng.choice([2, 4, 26]))
        t = synth.partial_dfa(Q, A, 0.2, seed, np.uint16) if seed % 2 else synth.random_dfa(Q, A, seed, np.uint16)
        x = rng.integers(0, A, 5000).astype(np.uint8)
        b = oracle.grid_boundaries(x.size, int(rng.choice([7, 100, 999])))
        assert oracle.lookback_stats(t, x, b, 1) == oracle.route_stats(t, x, b)


def test_lookback_brute_force_monotone_and_sound():
    """Python set iteration on tiny DFAs; |R^(k)| never grows with k; the true boundary
    state is always a candidate (soundness)."""
    rng = np.random.default_rng(5)
    for seed in range(6):
        Q, A = 6, 3
        t = synth.random_dfa(Q, A, seed, np.uint16).reshape(Q, A)
        x = rng.integers(0, A, 400).astype(np.uint8)
        b = oracle.grid_boundaries(x.size, 37)
        true = oracle.states_at(t, 0, x, b[1:-1])
        prev = None
        for k in (1, 2, 3, 5, 50):
            routes, steps = oracle.lookback_stats(t, x, b, k)
            want_r, want_s = 1, b[1] - b[0]
            for i in range(1, len(b) - 1):
                S = set(range(Q))
                for j in range(max(0, b[i] - k), b[i]):
                    S = {int(t[s, x[j]]) for s in S}
                assert int(true[i - 1]) in S
                want_r += len(S)
                want_s += len(S) * (b[i + 1] - b[i])
            assert (routes, steps) == (want_r, want_s)
            assert prev is None or routes <= prev
            prev = routes
