"""Pins for the Algorithm-1 model (oracle/alg1.py) and the route-count oracle:
Table I / Table II values, the "calculations" arithmetic, and the partition invariants."""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import alg1

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIGMA = "parel"
EXAMPLE = "plaraparallelapareparapl"


def sym(s):
    return [SIGMA.index(ch) for ch in s]


def table1():
    rows = [list(map(int, ln.split())) for ln in open(os.path.join(GOLD, "table1_parallel.txt"))
            if ln.strip() and not ln.startswith("#")]
    return np.array([r[1:] for r in rows], dtype=np.uint32)


def test_kmp_builder_reproduces_table1():
    """All 45 entries of Table I = KMP automaton of "parallel" over p,a,r,e,l."""
    t = synth.kmp_dfa(sym("parallel"), 5, np.uint32)
    assert t.shape == (9, 5)
    assert np.array_equal(t, table1())


def test_chunking_of_worked_example():
    """P0="plarap", P1="aralle", P2="lapare", P3="parapl"."""
    ch = alg1.chunk_input(sym(EXAMPLE), 4)
    assert ["".join(SIGMA[c] for c in x) for x in ch] == ["plarap", "aralle", "lapare", "parapl"]


def test_S_and_L_sets_of_example():
    """S = Q for a dense table; L on 'e' = {0,7} (yellow cells);
    P:193: L on 'l' = {0,5,6,8}; Table II P1: L on 'p' = {1}."""
    Tt = table1()
    assert alg1.S_set(Tt, SIGMA.index("l")) == set(range(9))
    assert alg1.L_set(Tt, SIGMA.index("e")) == {0, 7}
    assert alg1.L_set(Tt, SIGMA.index("l")) == {0, 5, 6, 8}
    assert alg1.L_set(Tt, SIGMA.index("p")) == {1}


def test_table2_routes():
    """Table II: R sets and visited states of every route (reading C6 adds
    the rule-implied route 7 on P3)."""
    Tt = table1()
    run = alg1.run_parem(Tt, 0, {8}, sym(EXAMPLE), 4)
    rows = [ln.split() for ln in open(os.path.join(GOLD, "table2_parem.txt"))
            if ln.strip() and not ln.startswith("#")]
    want_R = {}
    for r in rows:
        i = int(r[0][1:])
        want_R.setdefault(i, []).append(int(r[1]))
        assert run.routes[i][int(r[1])].visited == [int(x) for x in r[2:8]], r
    assert run.R == [sorted(want_R[i]) for i in range(4)] == [[0], [1], [0, 7], [0, 7]]
    # hits per route (F = {8}): only P2's route from 7 passes through 8
    assert run.routes[2][7].hits == 1 and run.routes[2][0].hits == 0
    assert (run.final_state, run.accepted, run.match_count) == (0, False, 1)


def test_calculation_counts():
    """P:193 / P:431: PaREM "five calculations" (= distinct states after the first
    symbol, reading C6; the raw rule count is 6), Enum 3*9+1 = 28, the all-'l' worst case
    3*4+1 = 13 and the 2.15 improvement."""
    Tt = table1()
    run = alg1.run_parem(Tt, 0, {8}, sym(EXAMPLE), 4)
    assert run.calculations == 6
    assert run.distinct_after_first == 5
    en = alg1.run_parem(Tt, 0, {8}, sym(EXAMPLE), 4, enum=True)
    assert en.calculations == 3 * 9 + 1 == 28
    assert (en.final_state, en.match_count) == (run.final_state, run.match_count)
    worst = 3 * len(alg1.L_set(Tt, SIGMA.index("l"))) + 1
    assert worst == 13 and round(28 / worst, 2) == 2.15
    # the C route-count oracle agrees with the model on the same partition
    assert oracle.route_stats(Tt, sym(EXAMPLE), [0, 6, 12, 18, 24]) == (6, 36)


def test_enum_hidden_table():
    """The hidden Enum table: all 28 routes of the General Enumeration
    Approach on the worked example, visited state by visited state; the two rows the paper
    misprints (reading C18) are checked against Table I directly."""
    Tt = table1()
    en = alg1.run_parem(Tt, 0, {8}, sym(EXAMPLE), 4, enum=True)
    rows = [ln.split() for ln in open(os.path.join(GOLD, "table_enum_hidden.txt"))
            if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 28 == en.calculations                       # "28 calculations"
    assert en.R == [[0]] + [list(range(9))] * 3
    typos = 0
    for r in rows:
        i, start, printed = int(r[0][1:]), int(r[1]), [int(x) for x in r[2:8]]
        got = en.routes[i][start].visited
        if r[-1] == "typo":
            typos += 1
            assert got[1:] == printed[1:] and printed[0] == 8
            assert got[0] == Tt[start][SIGMA.index("l")] == 0     # Table I: delta(2|3, l) = 0
        else:
            assert got == printed, r
    assert typos == 2
    # every route of P2 from a start other than 7 misses the match that 7 -> 8 makes
    assert [s for s in range(9) if en.routes[2][s].hits] == [7]


def test_compose_pins():
    """compose(P0, P1) maps 0 -> (7, 0); identity of an empty segment."""
    Tt = table1()
    ch = alg1.chunk_input(sym(EXAMPLE), 4)
    s0 = alg1.summary(Tt, {8}, ch[0], [0])
    s1 = alg1.summary(Tt, {8}, ch[1], [1])
    assert alg1.compose(s0, s1) == {0: (7, 0)}
    ident = {q: (q, 0) for q in range(9)}
    assert alg1.compose(s0, ident) == s0


def random_case(rng, partial):
    Q = int(rng.integers(1, 12))
    A = int(rng.integers(1, 5))
    seed = int(rng.integers(0, 1 << 30))
    t = synth.partial_dfa(Q, A, 0.1, seed) if partial else synth.random_dfa(Q, A, seed)
    F = set(np.nonzero(rng.random(Q) < 0.3)[0].tolist())
    q0 = int(rng.integers(0, Q))
    T = rng.integers(0, A, int(rng.integers(0, 200))).astype(np.uint8).tolist()
    return t, q0, F, T


@pytest.mark.parametrize("seed", range(40))
def test_engine_agreement_and_soundness(seed):
    """sequential = PaREM = Enum for every p, partial tables included;
    speculation soundness (true boundary state in R_i) on complete tables;
    routes_parem <= routes_enum."""
    rng = np.random.default_rng(seed)
    t, q0, F, T = random_case(rng, partial=seed % 3 == 0)
    Q = t.shape[0]
    acc = np.zeros(Q, dtype=bool)
    acc[list(F)] = True
    ref = oracle.walk(t, q0, acc, T)
    for p in (1, 2, 3, 5, 7, 16):
        run = alg1.run_parem(t, q0, F, T, p)
        en = alg1.run_parem(t, q0, F, T, p, enum=True)
        fin = oracle.DEAD if run.final_state == alg1.DEAD else run.final_state
        assert (fin, run.accepted, run.match_count) == (ref.final_state, ref.accepted, ref.match_count)
        assert (en.final_state, en.match_count) == (run.final_state, run.match_count)
        assert run.calculations <= en.calculations
        if p == 1:
            assert run.calculations == 1
        if seed % 3 and T:      # complete table: soundness of R = S n L
            bnd = np.cumsum([0] + [len(c) for c in run.chunks])[:-1]
            st = oracle.states_at(t, q0, T, bnd)
            for i in range(1, len(run.chunks)):
                assert int(st[i]) in run.R[i]
        if T:
            b = list(np.cumsum([0] + [len(c) for c in run.chunks]))
            assert oracle.route_stats(t, T, b)[0] == run.calculations


@pytest.mark.parametrize("seed", range(10))
def test_compose_associative(seed):
    rng = np.random.default_rng(1000 + seed)
    Q = int(rng.integers(1, 10))

    def rand_summary():
        return {q: (int(rng.integers(-1, Q)), int(rng.integers(0, 5))) for q in range(Q)}

    a, b, c = rand_summary(), rand_summary(), rand_summary()
    assert alg1.compose(alg1.compose(a, b), c) == alg1.compose(a, alg1.compose(b, c))


def test_kmp_L_closed_form():
    """For a KMP automaton L(c) = {j >= 1 : P[j-1] = c} u ({0} if c != P[0]), hence
    sum_c |L(c)| = |P| + |Sigma| - 1 (12 for "parallel", 4 for "abb", 15 for 12-mers
    over 4 symbols -- the cfg2 W_grid = 15/4)."""
    for P, A in ((sym("parallel"), 5), ([0, 1, 1], 2)):
        t = synth.kmp_dfa(P, A, np.uint32)
        for c in range(A):
            want = {j for j in range(1, len(P) + 1) if P[j - 1] == c} | ({0} if c != P[0] else set())
            assert alg1.L_set(t, c) == want
        assert sum(len(alg1.L_set(t, c)) for c in range(A)) == len(P) + A - 1
    P = synth.cfg2_pattern()
    t = synth.kmp_dfa(P, 4, np.uint16)
    assert sum(len(alg1.L_set(t, c)) for c in range(4)) == 15
