"""NEXT-3 front end (parem_regex_compile, host code in the library): the paper's RE language
(Table III) -> minimal DFA.  Pinned against the paper's own automaton (Table I),
the textbook (a|b)*abb DFA (reading C14), known minimal sizes, and brute force against
Python's `re` on every short string; a GPU test matches compiled patterns on the device."""
import itertools
import re

import numpy as np
import pytest

import oracle
import synth

GOLDEN_T1 = "tests/golden/table1_parallel.txt"


@pytest.fixture(scope="module")
def P():
    import paper_1412_1741_b200 as P

    P.lib()
    return P


def accepts(r, word_ids):
    s = r.start
    for c in word_ids:
        s = int(r.table[s, c])
    return bool(r.accept[s])


def test_abb_is_the_textbook_dfa(P):
    """(a|b)*abb over {a, b}: the minimal DFA in breadth-first numbering is exactly the KMP
    table of reading C14 (cfg1)."""
    r = P.compile_regex("(a|b)*abb", "ab")
    assert r.table.tolist() == [[1, 0], [1, 2], [1, 3], [1, 0]]
    assert r.accept.tolist() == [False, False, False, True] and r.start == 0


def test_parallel_search_is_table_I(P):
    """Sigma* parallel over (p, a, r, e, l): exactly Table I, accepting {8}."""
    r = P.compile_regex("parallel", "parel", search=True)
    rows = [list(map(int, ln.split())) for ln in open(GOLDEN_T1) if ln.strip() and not ln.startswith("#")]
    assert r.table.tolist() == [row[1:] for row in rows]
    assert r.accept.nonzero()[0].tolist() == [8]


@pytest.mark.parametrize("pat,alpha,Q", [
    ("(a|b)*a(a|b)(a|b)", "ab", 8),      # 2^3 classes: the classic subset-construction blow-up
    ("(a|b)*a(a|b)(a|b)(a|b)", "ab", 16),
    ("a*", "a", 1),
    ("a+", "a", 2),
    ("a?", "a", 3),                    # start (acc), after a (acc), trap
    ("", "ab", 2),                     # epsilon: start (acc) + trap
    ("[0..9]+", "0123456789", 2),
    ("(ab|c)*", "abc", 3),             # Table III's group example
])
def test_minimal_sizes(P, pat, alpha, Q):
    assert len(P.compile_regex(pat, alpha).table) == Q


def test_paper_ast_example_alphabet(P):
    """Fig. 4's (a|b)?c*[0..3]b+ (P:249): default alphabet = the pattern's bytes, range
    expanded over it."""
    r = P.compile_regex("(a|b)?c*[0..3]b+")
    assert r.alphabet == b"0123abc"
    py = re.compile(r"(a|b)?c*[0-3]b+")
    for n in range(6):
        for w in itertools.product(range(7), repeat=n):
            s = "".join(chr(r.alphabet[c]) for c in w)
            assert accepts(r, w) == bool(py.fullmatch(s)), s


@pytest.mark.parametrize("bad", ["(ab", "a)", "[a..]", "[b..a]", "x", "*a", "a|(b", "\\"])
def test_syntax_errors(P, bad):
    with pytest.raises(P.ParemError):
        P.compile_regex(bad, "ab")


def rand_re(rng, depth, alpha):
    """Random RE over `alpha` in both syntaxes: (ours, Python)."""
    k = int(rng.integers(0, 7 if depth > 0 else 2))
    if k == 0 or depth == 0:
        c = alpha[int(rng.integers(0, len(alpha)))]
        return c, c
    if k == 1:
        lo, hi = sorted(rng.choice(list(alpha), 2))
        return f"[{lo}..{hi}]", f"[{lo}-{hi}]"
    a, pa = rand_re(rng, depth - 1, alpha)
    if k == 2:
        b, pb = rand_re(rng, depth - 1, alpha)
        return a + b, pa + pb
    if k == 3:
        b, pb = rand_re(rng, depth - 1, alpha)
        return f"({a}|{b})", f"({pa}|{pb})"
    op = "*+?"[k - 4]
    return f"({a}){op}", f"({pa}){op}"


@pytest.mark.parametrize("seed", range(40))
def test_random_regex_brute_force(P, seed):
    """Anchored and search compilations against Python's `re` on every string up to
    length 6 over {a, b, c} (search: count of end positions of some occurrence)."""
    rng = np.random.default_rng(seed)
    ours, py = rand_re(rng, 4, "abc")
    rx = re.compile(py)
    r = P.compile_regex(ours, "abc")
    s = P.compile_regex(ours, "abc", search=True)
    for n in range(7):
        for w in itertools.product(range(3), repeat=n):
            text = "".join("abc"[c] for c in w)
            assert accepts(r, w) == bool(rx.fullmatch(text)), (ours, text)
    for _ in range(20):
        w = rng.integers(0, 3, int(rng.integers(0, 30)))
        text = "".join("abc"[c] for c in w)
        want = sum(any(rx.fullmatch(text[j:k]) for j in range(k + 1)) for k in range(1, len(text) + 1))
        got = oracle.walk(s.table, s.start, s.accept, w.astype(np.uint8)).match_count
        assert got == want, (ours, text)


@pytest.mark.gpu
@pytest.mark.parametrize("pat,alpha", [("parallel", "parel"), ("(a|b)*abb", "ab"), ("(ACG|T)+A?[C..G]", "ACGT"),
                                       ("x[0..9]+y", "0123456789xyz")])
def test_regex_on_gpu(P, cuda_device, pat, alpha):
    """Compiled patterns matched on the device agree with the oracle (search automaton)."""
    import torch

    r = P.compile_regex(pat, alpha, search=True)
    x = synth.uniform_symbols((1 << 20) + 5, len(r.alphabet), seed=len(pat))
    ref = oracle.walk(r.table, r.start, r.accept, x)
    with P.Dfa(r.table, r.start, r.accept) as d:
        got = d.match(torch.from_numpy(x).to("cuda"))
    assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)


# ---------------------------------------------------------------- transition-table text I/O
def test_table_text_table_I_layout(P):
    """Table I as the log file of P:314 in SPEC's layout: header
    `symbols p a r e l`, `start 0`, `finals 8`, nine rows; the text reads back exactly."""
    r = P.compile_regex("parallel", "parel", search=True)
    txt = P.table_to_text(r.table, r.start, r.accept, r.alphabet)
    lines = txt.split("\n")
    assert lines[0] == "symbols\tp\ta\tr\te\tl" and lines[1] == "start\t0" and lines[2] == "finals\t8"
    assert len(lines) == 3 + 9 + 1 and lines[-1] == ""
    assert lines[3 + 5] == "5\t1\t0\t0\t0\t6" and lines[3 + 7] == "7\t1\t0\t0\t0\t8"   # delta(5,l)=6, delta(7,l)=8
    back = P.table_from_text(txt)
    assert back.table.tolist() == r.table.tolist() and back.start == r.start
    assert back.accept.tolist() == r.accept.tolist() and back.alphabet == r.alphabet


@pytest.mark.parametrize("seed", range(20))
def test_table_text_round_trip_random(P, seed):
    """Round trip is the identity: random partial DFAs (DEAD entries as '-'), any
    alphabet bytes (escaped when not printable), zero or many finals, u16 and u32 tables."""
    rng = np.random.default_rng(seed)
    Q, A = int(rng.integers(1, 60)), int(rng.integers(1, 40))
    dt = np.uint16 if seed % 2 else np.uint32
    t = synth.partial_dfa(Q, A, 0.3, seed, dt)
    acc = rng.random(Q) < (0.0 if seed % 5 == 0 else 0.4)
    alphabet = bytes(rng.permutation(256)[:A].astype(np.uint8))
    start = int(rng.integers(0, Q))
    txt = P.table_to_text(t, start, acc, alphabet)
    back = P.table_from_text(txt)
    want = np.where(t == np.iinfo(dt).max, 0xFFFFFFFF, t.astype(np.int64))
    assert back.table.astype(np.int64).tolist() == want.tolist()
    assert (back.start, back.accept.tolist(), back.alphabet) == (start, acc.tolist(), alphabet)
    assert P.table_to_text(back.table, back.start, back.accept, back.alphabet) == txt


@pytest.mark.parametrize("text,line", [
    ("", 1), ("symbol\ta\nstart\t0\nfinals\n0\t0\n", 1), ("symbols\ta\ta\nstart\t0\nfinals\n0\t0\t0\n", 1),
    ("symbols\ta\nstar\t0\nfinals\n0\t0\n", 2), ("symbols\ta\nstart\t5\nfinals\n0\t0\n", 2),
    ("symbols\ta\nstart\t0\nfinals\t3\n0\t0\n", 3), ("symbols\ta\nstart\t0\nfinals\n1\t0\n", 4),
    ("symbols\ta\tb\nstart\t0\nfinals\n0\t0\n", 4), ("symbols\ta\nstart\t0\nfinals\n0\t0\n1\t7\n", 5),
    ("symbols\ta\nstart\t0\nfinals\n0\tx\n", 4), ("symbols\ta\nstart\t0\nfinals\n", 4),
])
def test_table_text_parse_errors_name_the_line(P, text, line):
    with pytest.raises(P.ParemError) as ei:
        P.table_from_text(text)
    assert f"line {line}:" in str(ei.value), str(ei.value)


def test_table_text_loaded_table_matches_like_the_original(P):
    """A table written and read back drives the oracle to the same result (the pipeline of
    S:437 without the GPU): Table I on the paper's worked input, count 1."""
    r = P.compile_regex("parallel", "parel", search=True)
    back = P.table_from_text(P.table_to_text(r.table, r.start, r.accept, r.alphabet))
    x = back.encode(b"plaraparallelapareparapl")
    ref = oracle.walk(back.table, back.start, back.accept, x)
    assert (ref.final_state, ref.match_count) == (0, 1)
