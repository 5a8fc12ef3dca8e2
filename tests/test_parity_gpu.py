"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element
on the same seeded inputs -- final state, accept flag and match count bit-exact (integer
path, BASELINE north_star), stats against the paper's route rule (oracle.route_stats)."""
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


def to_dev(torch, x, offset=0):
    """Copy bytes to the device; ``offset`` > 0 yields a deliberately unaligned view."""
    buf = torch.empty(x.size + offset + 16, dtype=torch.uint8, device="cuda")
    view = buf[offset:offset + x.size]
    if x.size:
        view.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return view


def check(parem, torch, table, start, acc, x, opts=None, offset=0, expect=None):
    ref = oracle.walk(table, start, acc, x)
    with parem.Dfa(table, start, acc) as d:
        got = d.match(to_dev(torch, x, offset), opts)
    if ref.status == oracle.ESYMBOL:
        assert got.status == parem.PAREM_ESYMBOL and got.bad_offset == ref.bad_offset, (got, ref)
        return got
    assert got.status == 0, got
    assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count), \
        (got, ref, table.shape, x.size, opts and (opts.chunk_len, opts.boundary_policy, opts.candidates, opts.kernel))
    return got


# ---------------------------------------------------------------- configs, CI-sized
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [1 << 20, (1 << 20) + 13])
def test_configs_small(parem, torch_mod, k, n):
    c = synth.config(k, n=n)
    x = c.make_input()
    check(parem, torch_mod, c.table, c.start, c.accept, x)


# ---------------------------------------------------------------- random DFAs
def rand_dfa(rng, Q, A, partial):
    seed = int(rng.integers(0, 1 << 30))
    dt = np.uint16 if rng.random() < 0.6 else np.uint32
    t = synth.partial_dfa(Q, A, float(rng.choice([0.02, 0.1, 0.4])), seed, dt) if partial else \
        synth.random_dfa(Q, A, seed, dt)
    acc = rng.random(Q) < float(rng.choice([0.05, 0.3, 0.9]))
    return t, int(rng.integers(0, Q)), acc


SIZES = [0, 1, 2, 15, 16, 17, 255, 1000, 4097, 65539]


@pytest.mark.parametrize("seed", range(120))
def test_random_dfas(parem, torch_mod, seed):
    rng = np.random.default_rng(seed)
    Q = int(rng.choice([1, 2, 3, 5, 13, 31, 32, 33, 100, 256, 1024]))
    A = int(rng.choice([1, 2, 3, 4, 5, 26, 256]))
    t, q0, acc = rand_dfa(rng, Q, A, partial=seed % 4 == 0)
    for n in rng.choice(SIZES, 3, replace=False):
        n = int(n)
        x = rng.integers(0, A, n).astype(np.uint8)
        opts = parem.options(chunk_len=int(rng.choice([0, 1, 3, 16, 100, 4096])),
                             boundary=str(rng.choice(["grid", "snap"])),
                             candidates=str(rng.choice(["parem", "parem", "enum"])))
        check(parem, torch_mod, t, q0, acc, x, opts, offset=int(rng.integers(0, 16)))


@pytest.mark.parametrize("kernel", ["tiny", "lanes"])
@pytest.mark.parametrize("seed", range(30))
def test_both_kernels_agree(parem, torch_mod, kernel, seed):
    """The lanes kernel also handles small DFAs when forced (DFAs <= 32 states have a lanes
    table only when > 32 states, so the tiny case forces only where allowed)."""
    rng = np.random.default_rng(5000 + seed)
    Q = int(rng.choice([2, 7, 13, 30])) if kernel == "tiny" else int(rng.choice([40, 300, 2000]))
    A = int(rng.choice([2, 4, 26, 256]))
    t, q0, acc = rand_dfa(rng, Q, A, partial=seed % 3 == 0)
    n = int(rng.integers(1, 200000))
    x = rng.integers(0, A, n).astype(np.uint8)
    check(parem, torch_mod, t, q0, acc, x, parem.options(kernel=kernel), offset=seed % 16)


@pytest.mark.parametrize("L", [1, 2, 3, 7, 16, 17, 64, 1000])
def test_forced_chunk_lengths_kmp(parem, torch_mod, L):
    """Chunking invariance on the DNA-motif DFA: any chunk length composes to the
    sequential result, with both boundary policies."""
    P = synth.cfg2_pattern()
    t = synth.kmp_dfa(P, 4, np.uint16)
    acc = np.zeros(13, dtype=bool)
    acc[12] = True
    rng = np.random.default_rng(L)
    x = rng.integers(0, 4, 20000).astype(np.uint8)
    for pos in rng.integers(0, 20000 - 12, 50):
        x[pos:pos + 12] = P
    for b in ("grid", "snap"):
        got = check(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=L, boundary=b))
        assert got.match_count >= 40


# ---------------------------------------------------------------- stats vs the paper's rule
@pytest.mark.parametrize("k,L", [(1, 64), (2, 256), (2, 1000), (3, 4096), (5, 8192)])
def test_route_stats_grid(parem, torch_mod, k, L):
    """routes = sum_i |R_i| and route_steps = sum_i |R_i| len_i for the grid partition,
    computed by the oracle directly from R_i = S(T[b_i]) n L(T[b_i - 1])."""
    c = synth.config(k, n=300000)
    x = c.make_input()
    with parem.Dfa(c.table, c.start, c.accept) as d:
        got = d.match(to_dev(torch_mod, x), parem.options(chunk_len=L, boundary="grid"))
    b = oracle.grid_boundaries(x.size, L)
    assert got.num_chunks == len(b) - 1
    assert (got.routes, got.route_steps) == oracle.route_stats(c.table, x, b)


def test_route_stats_partial_and_enum(parem, torch_mod):
    rng = np.random.default_rng(77)
    t = synth.partial_dfa(20, 4, 0.3, 77, np.uint16)
    acc = rng.random(20) < 0.3
    x = rng.integers(0, 4, 50000).astype(np.uint8)
    with parem.Dfa(t, 3, acc) as d:
        xd = to_dev(torch_mod, x)
        got = d.match(xd, parem.options(chunk_len=97, boundary="grid"))
        b = oracle.grid_boundaries(x.size, 97)
        assert (got.routes, got.route_steps) == oracle.route_stats(t, x, b)
        en = d.match(xd, parem.options(chunk_len=97, boundary="grid", candidates="enum"))
        p = len(b) - 1
        assert en.routes == 1 + (p - 1) * 20            # (p-1)|Q| + 1
        assert (en.final_state, en.match_count) == (got.final_state, got.match_count)


def test_snap_reduces_work(parem, torch_mod):
    c = synth.config(2, n=1 << 22)
    x = c.make_input()
    with parem.Dfa(c.table, 0, c.accept) as d:
        xd = to_dev(torch_mod, x)
        g = d.match(xd, parem.options(chunk_len=4096, boundary="grid"))
        s = d.match(xd, parem.options(chunk_len=4096, boundary="snap"))
    assert g.num_chunks == s.num_chunks
    W_grid, W_exec = g.route_steps / x.size, s.route_steps / x.size
    assert abs(W_grid - 3.75) < 0.05          # 15/4 for any 12-mer (closed form)
    assert W_exec < 2.05                      # min_c |L(c)| = 2 for the seed-2 pattern
    assert (g.final_state, g.match_count) == (s.final_state, s.match_count)


# ---------------------------------------------------------------- edge cases
def test_empty_input(parem, torch_mod):
    for acc0 in (False, True):
        acc = np.array([acc0, False])
        t = np.array([[1, 0], [0, 1]], dtype=np.uint16)
        check(parem, torch_mod, t, 0, acc, np.zeros(0, np.uint8))


@pytest.mark.parametrize("Q,A", [(4, 2), (13, 4), (9, 5), (256, 26), (1024, 256)])
def test_symbol_errors_smallest_offset(parem, torch_mod, Q, A):
    rng = np.random.default_rng(Q * A)
    t = synth.random_dfa(Q, A, 3, np.uint16)
    acc = rng.random(Q) < 0.2
    if A == 256:
        pytest.skip("every byte is a valid symbol")
    for trial in range(4):
        x = rng.integers(0, A, 100000).astype(np.uint8)
        bad = np.sort(rng.integers(0, x.size, 3))
        x[bad] = rng.integers(A, 256, 3)
        got = check(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=int(rng.choice([0, 5, 300]))))
        assert got.status == parem.PAREM_ESYMBOL and got.bad_offset == bad[0]


def test_dead_semantics_counterexample(parem, torch_mod):
    """C9: delta(1,a) = DEAD; "aa" must die at the chunk boundary even when R_1 = {} ."""
    t = np.array([[1, 0], [0xFFFF, 0]], dtype=np.uint16)
    acc = np.array([False, True])
    for x in ([0, 0], [0, 0, 1, 1, 0], [1, 0, 1, 0, 0, 1]):
        for L in (1, 2, 3):
            check(parem, torch_mod, t, 0, acc, np.array(x, np.uint8), parem.options(chunk_len=L))


def test_worked_example_table2(parem, torch_mod):
    """The paper's worked example (Table II): count 1, final 0, 4 chunks of 6."""
    t = synth.kmp_dfa([0, 1, 2, 1, 4, 4, 3, 4], 5, np.uint32)
    acc = np.zeros(9, dtype=bool)
    acc[8] = True
    x = np.array(["parel".index(ch) for ch in "plaraparallelapareparapl"], np.uint8)
    got = check(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=6, boundary="grid"))
    assert (got.final_state, got.match_count, got.num_chunks, got.routes) == (0, 1, 4, 6)
    en = check(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=6, boundary="grid", candidates="enum"))
    assert en.routes == 28


# ---------------------------------------------------------------- async / continue / host
def test_async_continue_and_host(parem, torch_mod):
    torch = torch_mod
    c = synth.config(3, n=3_000_017)
    x = c.make_input()
    ref = oracle.walk(c.table, c.start, c.accept, x)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        xd = to_dev(torch, x)
        ws = torch.empty(d.workspace_bytes(x.size), dtype=torch.uint8, device="cuda")
        res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        d.match_async(xd, ws, res)
        got = parem.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
        assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)
        # streaming: three segments with carried state
        cuts = [0, 1_000_003, 2_000_000, x.size]
        ws2 = torch.empty(d.workspace_bytes(x.size), dtype=torch.uint8, device="cuda")
        for i in range(3):
            seg = xd[cuts[i]:cuts[i + 1]]
            d.match_continue_async(seg, cuts[i], ws2, res if i else None, res)
        got = parem.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
        assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)
        h = torch.from_numpy(x).pin_memory()
        got = d.match_host(h)
        assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)


def test_host_path_symbol_error_offset(parem, torch_mod):
    c = synth.config(2, n=(64 << 20) + 1000)
    x = c.make_input()
    x[(64 << 20) + 17] = 9        # in the second 64 MiB segment
    with parem.Dfa(c.table, 0, c.accept) as d:
        got = d.match_host(x)
    assert got.status == parem.PAREM_ESYMBOL and got.bad_offset == (64 << 20) + 17


# ---------------------------------------------------------------- full BASELINE sizes
@pytest.mark.slow
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_configs_full_size(parem, torch_mod, k):
    """BASELINE.json configs at full size, default (bench) launch configuration,
    bit-exact against the single-threaded oracle."""
    c = synth.config(k)
    x = c.make_input()
    ref = oracle.walk(c.table, c.start, c.accept, x)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        xd = torch_mod.from_numpy(x).to("cuda")
        got = d.match(xd)
    assert got.status == 0
    assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)


@pytest.mark.slow
@pytest.mark.parametrize("k,cap", [(1, None), (2, None), (3, 1 << 24)])
def test_find_positions_full_size(parem, torch_mod, k, cap):
    """NEXT-4 at full BASELINE size, default launch configuration: the match end offsets of
    parem_find_async equal the oracle's element by element (every position for cfg1 / cfg2;
    the first 2^24 of cfg3's ~5e8, whose total count must match too)."""
    c = synth.config(k)
    x = c.make_input()
    want, total = oracle.positions(c.table, c.start, c.accept, x, cap)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        r, pos = d.find(torch_mod.from_numpy(x).to("cuda"), max_positions=cap)
    assert r.status == 0 and r.match_count == total
    got = pos.cpu().numpy().astype(np.uint64)
    assert got.size == want.size and np.array_equal(got, want)


# ---------------------------------------------------------------- route merging stress
@pytest.mark.parametrize("Q", [3, 5, 13, 31])
def test_permutation_dfa_routes_never_merge(parem, torch_mod, Q):
    """delta(q, c) = (q + c + 1) mod Q: every column is a permutation (|L(c)| = Q, the
    paper's worst case P:70), so a chunk's routes never converge."""
    A = 4
    t = np.array([[(q + c + 1) % Q for c in range(A)] for q in range(Q)], dtype=np.uint16)
    acc = np.zeros(Q, dtype=bool)
    acc[Q // 2] = True
    x = synth.uniform_symbols((1 << 20) + 33, A, seed=Q)
    for b in ("snap", "grid"):
        check(parem, torch_mod, t, 1, acc, x, parem.options(boundary=b))


@pytest.mark.parametrize("p_reset", [1e-4, 1e-3, 2e-2])
def test_partially_merging_warps(parem, torch_mod, p_reset):
    """A mod-Q counter with a rare reset symbol: chunks that contain a reset merge their
    routes, the others do not -- lanes of one warp disagree."""
    Q, A = 11, 4
    t = np.array([[(q + 1) % Q if c < 3 else 0 for c in range(A)] for q in range(Q)], dtype=np.uint16)
    acc = np.zeros(Q, dtype=bool)
    acc[[0, 7]] = True
    rng = np.random.default_rng(int(1 / p_reset))
    x = rng.integers(0, 3, 4 << 20).astype(np.uint8)
    x[rng.random(x.size) < p_reset] = 3
    for b in ("grid", "snap"):
        for L in (0, 4096, 8192 + 64):
            check(parem, torch_mod, t, 0, acc, x, parem.options(boundary=b, chunk_len=L))


# ---------------------------------------------------------------- converging path (kernel 3)
@pytest.mark.parametrize("k", [3, 4, 5])
@pytest.mark.parametrize("L", [0, 16, 333, 4096, 100000])
def test_conv_configs(parem, torch_mod, k, L):
    """Set walk + follow + join + heads (kernels_conv.cu) against the oracle, for chunk
    lengths from tiny (every chunk open: the join walks them all) to long (anchors), with
    both candidate rules and an unaligned input view."""
    c = synth.config(k, n=(1 << 20) + 7)
    x = c.make_input()
    for cand in ("parem", "enum"):
        got = check(parem, torch_mod, c.table, c.start, c.accept, x,
                    parem.options(chunk_len=L, kernel="conv", candidates=cand), offset=(L + k) % 16)
        if cand == "parem" and L:
            b = oracle.grid_boundaries(x.size, L)
            assert got.num_chunks == len(b) - 1
            assert (got.routes, got.route_steps) == oracle.route_stats(c.table, x, b)
        if cand == "parem" and L >= 4096:
            # executed lookups (parem_result.lookups_k, units of 1024): every byte is walked at
            # least once (set walk or follow), and merging never costs more than walking every
            # candidate over its whole chunk (the paper's route_steps) plus the join's head walks
            assert x.size <= got.lookups <= got.route_steps + 32 * x.size, got
            assert got.lookups < got.route_steps // 4, got   # routes merge early on these DFAs


@pytest.mark.parametrize("seed", range(40))
def test_conv_random_dfas(parem, torch_mod, seed):
    """Random complete DFAs (33..2000 states, any alphabet) on the converging path, with
    random chunk lengths and start states; start states may be accepting."""
    rng = np.random.default_rng(9000 + seed)
    Q = int(rng.choice([33, 40, 100, 256, 600, 2000]))
    A = int(rng.choice([2, 3, 4, 26, 200, 256]))
    t = synth.random_dfa(Q, A, int(rng.integers(0, 1 << 30)), np.uint16 if seed % 2 else np.uint32)
    acc = rng.random(Q) < float(rng.choice([0.05, 0.5, 0.95]))
    q0 = int(rng.integers(0, Q))
    with parem.Dfa(t, q0, acc) as d:
        if d.plan(1 << 20)["kernel"] != 3:
            pytest.skip("routes of this DFA do not merge within the probe")
    n = int(rng.choice([1, 17, 4095, 100003, 1 << 20]))
    x = rng.integers(0, A, n).astype(np.uint8)
    L = int(rng.choice([0, 0, 1, 50, 1000, 30000]))
    check(parem, torch_mod, t, q0, acc, x, parem.options(chunk_len=L, kernel="conv"), offset=seed % 16)


def test_conv_rejects_non_merging_dfa(parem, torch_mod):
    """A permutation DFA never merges routes: auto picks the lanes kernel and forcing the
    converging path is an EINVAL, not a wrong answer."""
    Q, A = 64, 4
    t = np.array([[(q + c + 1) % Q for c in range(A)] for q in range(Q)], dtype=np.uint16)
    acc = np.zeros(Q, dtype=bool)
    acc[5] = True
    with parem.Dfa(t, 0, acc) as d:
        assert d.plan(1 << 20)["kernel"] == 2
        with pytest.raises(parem.ParemError):
            d.match(to_dev(torch_mod, np.zeros(100, np.uint8)), parem.options(kernel="conv"))
    x = synth.uniform_symbols(300001, A, seed=64)
    check(parem, torch_mod, t, 0, acc, x)


def test_conv_symbol_errors(parem, torch_mod):
    """ESYMBOL with the smallest offset whether the bad byte sits in a head (K3) or a tail
    (K2) of the converging path."""
    c = synth.config(3, n=1 << 20)
    rng = np.random.default_rng(3)
    for L in (0, 64, 5000):
        for trial in range(3):
            x = c.make_input().copy()
            bad = np.sort(rng.integers(0, x.size, 2))
            x[bad] = 200
            got = check(parem, torch_mod, c.table, c.start, c.accept, x, parem.options(chunk_len=L, kernel="conv"))
            assert got.status == parem.PAREM_ESYMBOL and got.bad_offset == bad[0]


# ---------------------------------------------------------------- clean-workspace contract
@pytest.mark.parametrize("k,kernel", [(1, "auto"), (2, "auto"), (3, "conv"), (3, "lanes"), (5, "conv")])
def test_ws_clean_reuse(parem, torch_mod, k, kernel):
    """PAREM_FLAG_WS_CLEAN: a zero-filled workspace reused across calls without any reset --
    every completed call (ESYMBOL included) must leave the header zeroed for the next."""
    torch = torch_mod
    c = synth.config(k, n=300_007)
    rng = np.random.default_rng(k)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        opts = parem.options(kernel=kernel, ws_clean=True)
        ws = torch.zeros(d.workspace_bytes(c.n, opts), dtype=torch.uint8, device="cuda")
        res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        for trial in range(6):
            x = c.make_input().copy()
            if trial % 3 == 1 and c.A < 256:
                x[int(rng.integers(0, x.size))] = 255
            x = x[: x.size - 1000 * trial]
            ref = oracle.walk(c.table, c.start, c.accept, x)
            d.match_async(to_dev(torch, x), ws, res, opts)
            got = parem.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
            if ref.status == oracle.ESYMBOL:
                assert got.status == parem.PAREM_ESYMBOL and got.bad_offset == ref.bad_offset
            else:
                assert got.status == 0 and (got.final_state, got.accepted, got.match_count) == \
                    (ref.final_state, ref.accepted, ref.match_count), (trial, got, ref)
            assert not ws[:64].any(), "header not left zeroed"


def test_profile_records_kernels(parem, torch_mod):
    c = synth.config(3, n=1 << 20)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        xd = to_dev(torch_mod, c.make_input())
        parem.profile(True)
        d.match(xd)
        d.match(xd)
        parem.profile(False)
        recs = parem.profile_read()
    names = [r[1] for r in recs]
    assert names == ["conv_set", "conv_follow", "conv_ends", "conv_wide", "conv_map1", "conv_map", "conv_block",
                     "conv_super", "conv_path", "conv_blockin", "conv_resolve"] * 2
    assert {r[0] for r in recs} == {0, 1} and all(r[2] > 0 for r in recs)


# ---------------------------------------------------------------- NEXT-4: match positions
def check_find(parem, torch, table, start, acc, x, opts=None, cap=None, offset=0):
    pos_ref, cnt_ref = oracle.positions(table, start, acc, x, cap=cap)
    with parem.Dfa(table, start, acc) as d:
        r, pos = d.find(to_dev(torch, x, offset), max_positions=cap, opts=opts)
    assert r.status == 0 and r.match_count == cnt_ref, (r, cnt_ref)
    got = pos.cpu().numpy().astype(np.uint64)
    assert got.size == pos_ref.size and (got == pos_ref).all(), (got[:10], pos_ref[:10])
    return r


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_find_configs(parem, torch_mod, k):
    """Match end offsets on every BASELINE config (CI size, ragged tail): tiny, converging
    path; ascending, element by element against the oracle."""
    c = synth.config(k, n=(1 << 20) + 333)
    x = c.make_input()
    check_find(parem, torch_mod, c.table, c.start, c.accept, x)


@pytest.mark.parametrize("kernel,L,cand,boundary", [("auto", 0, "parem", "auto"), ("auto", 1000, "parem", "snap"),
                                                    ("auto", 64, "enum", "grid"), ("lanes", 0, "parem", "snap"),
                                                    ("lanes", 5000, "enum", "grid"), ("conv", 333, "parem", "grid")])
def test_find_options(parem, torch_mod, kernel, L, cand, boundary):
    c = synth.config(3 if kernel != "auto" else 2, n=700_001)
    x = c.make_input()
    check_find(parem, torch_mod, c.table, c.start, c.accept, x,
               parem.options(chunk_len=L, candidates=cand, boundary=boundary, kernel=kernel), offset=L % 16)


def test_find_caps_partial_and_paper_example(parem, torch_mod):
    """Caps keep the first offsets; partial tables stop at DEAD; the worked example's one
    occurrence of "parallel" ends at offset 12."""
    c = synth.config(2, n=1 << 20)
    x = c.make_input()
    for cap in (0, 1, 7, 50):
        check_find(parem, torch_mod, c.table, c.start, c.accept, x, cap=cap)
    rng = np.random.default_rng(5)
    for seed in range(6):
        t = synth.partial_dfa(int(rng.choice([5, 40, 300])), 4, 0.02, seed, np.uint16)
        acc = rng.random(t.shape[0]) < 0.4
        x = rng.integers(0, 4, 200_000).astype(np.uint8)
        check_find(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=int(rng.choice([0, 100]))))
    t = synth.kmp_dfa([0, 1, 2, 1, 4, 4, 3, 4], 5, np.uint32)
    acc = np.zeros(9, dtype=bool)
    acc[8] = True
    x = np.array(["parel".index(ch) for ch in "plaraparallelapareparapl"], np.uint8)
    r = check_find(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=6, boundary="grid"))
    with parem.Dfa(t, 0, acc) as d:
        _, pos = d.find(to_dev(torch_mod, x))
    assert pos.tolist() == [12] and r.match_count == 1


@pytest.mark.parametrize("k", [3, 4, 5])
@pytest.mark.parametrize("kind", ["zeros", "period3", "runs", "two_symbols"])
def test_conv_adversarial_inputs(parem, torch_mod, k, kind):
    """Inputs on which routes do NOT merge to <= 4 states inside a chunk (a repeated symbol
    keeps the cycle points of one column alive, short periods keep a few states apart):
    the join composes small maps in parallel instead of walking chunks one by one."""
    c = synth.config(k, n=1 << 20)
    rng = np.random.default_rng(k)
    n = (1 << 21) + 5
    if kind == "zeros":
        x = np.zeros(n, np.uint8)
    elif kind == "period3":
        x = np.resize(np.array([1, 2, 3], np.uint8), n)
    elif kind == "two_symbols":
        x = rng.integers(0, 2, n).astype(np.uint8)
    else:
        x = np.repeat(rng.integers(0, c.A, n // 1000 + 1).astype(np.uint8), 1000)[:n]
    for L in (0, 4096):
        check(parem, torch_mod, c.table, c.start, c.accept, x, parem.options(chunk_len=L, kernel="conv"))
    check_find(parem, torch_mod, c.table, c.start, c.accept, x, parem.options(kernel="conv"), cap=1000)


# ---------------------------------------------------------------- graphs and streams
@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_graph_capture_replay(parem, torch_mod, k):
    """parem_match_async is graph-capturable (tiny: one kernel; converging path: eight):
    a captured match replayed over new contents of the same input buffer stays exact
    (the clean-workspace contract holds across replays)."""
    torch = torch_mod
    c = synth.config(k, n=400_003)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        opts = parem.options(ws_clean=True)
        ws = torch.zeros(d.workspace_bytes(c.n, opts), dtype=torch.uint8, device="cuda")
        res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        xd = torch.empty(c.n, dtype=torch.uint8, device="cuda")
        xd.copy_(torch.from_numpy(c.make_input()))
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            d.match_async(xd, ws, res, opts, s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            d.match_async(xd, ws, res, opts, s)
        rng = np.random.default_rng(k)
        for rep in range(3):
            x = c.make_input() if rep == 0 else synth.uniform_symbols(c.n, c.A, seed=100 + rep)
            xd.copy_(torch.from_numpy(x))
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            got = parem.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
            ref = oracle.walk(c.table, c.start, c.accept, x)
            assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)


def test_concurrent_streams(parem, torch_mod):
    """One immutable DFA handle, two streams, two workspaces, different inputs in flight."""
    torch = torch_mod
    c = synth.config(3, n=1_000_003)
    xa, xb = c.make_input(), synth.uniform_symbols(c.n, c.A, seed=77)
    ra, rb = (oracle.walk(c.table, c.start, c.accept, x) for x in (xa, xb))
    with parem.Dfa(c.table, c.start, c.accept) as d:
        outs = []
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for x, s in zip((xa, xb), streams):
            ws = torch.zeros(d.workspace_bytes(c.n), dtype=torch.uint8, device="cuda")
            res = torch.zeros(64, dtype=torch.uint8, device="cuda")
            xd = to_dev(torch, x)
            torch.cuda.synchronize()
            outs.append((ws, res, xd))
        for i in range(4):
            for (ws, res, xd), s in zip(outs, streams):
                d.match_async(xd, ws, res, None, s)
        torch.cuda.synchronize()
        for (ws, res, xd), ref in zip(outs, (ra, rb)):
            got = parem.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
            assert (got.final_state, got.accepted, got.match_count) == (ref.final_state, ref.accepted, ref.match_count)


# ---------------------------------------------------------------- NEXT-2 (i): look-back candidates
@pytest.mark.parametrize("k_lb", [1, 2, 4, 16])
def test_lookback_candidates(parem, torch_mod, k_lb):
    """R_i = delta*(Q, T[b_i - k, b_i)) n S(T[b_i]) in the tiny kernel: results exact, and the
    GPU's routes / route_steps equal the oracle's look-back statistics (k = 1: the paper's)."""
    rng = np.random.default_rng(k_lb)
    cases = [(synth.config(1, n=200_003), None), (synth.config(2, n=300_001), None)]
    for k, cfg in enumerate(cases):
        c = cfg[0]
        x = c.make_input()
        for L in (64, 1000):
            got = check(parem, torch_mod, c.table, c.start, c.accept, x,
                        parem.options(chunk_len=L, boundary="grid", candidates="lookback", lookback=k_lb))
            b = oracle.grid_boundaries(x.size, L)
            assert (got.routes, got.route_steps) == oracle.lookback_stats(c.table, x, b, k_lb)
            if k_lb == 1:
                assert (got.routes, got.route_steps) == oracle.route_stats(c.table, x, b)
    for seed in range(6):
        Q, A = int(rng.choice([3, 9, 20, 31])), int(rng.choice([2, 4, 7]))
        t = synth.partial_dfa(Q, A, 0.1, seed, np.uint16) if seed % 2 else synth.random_dfa(Q, A, seed, np.uint16)
        acc = rng.random(Q) < 0.3
        x = rng.integers(0, A, 50_000).astype(np.uint8)
        got = check(parem, torch_mod, t, 0, acc, x, parem.options(chunk_len=97, boundary="grid",
                                                                 candidates="lookback", lookback=k_lb))
        assert (got.routes, got.route_steps) == oracle.lookback_stats(t, x, oracle.grid_boundaries(x.size, 97), k_lb)
        check(parem, torch_mod, t, 0, acc, x, parem.options(candidates="lookback", lookback=k_lb))   # planner + SNAP/AUTO


def test_lookback_rejected_off_tiny(parem, torch_mod):
    c = synth.config(3, n=1000)
    with parem.Dfa(c.table, c.start, c.accept) as d:
        with pytest.raises(parem.ParemError):
            d.match(to_dev(torch_mod, c.make_input()), parem.options(candidates="lookback", lookback=4))
        with pytest.raises(parem.ParemError):
            d.match(to_dev(torch_mod, c.make_input()), parem.options(candidates="lookback"))


def test_conv_wide_chunks(parem, torch_mod):
    """Chunks whose candidate set never shrinks to 32 states ("wide"): symbol 0 permutes the
    64 states (a rotation), symbols 1..3 are random maps, so the DFA converges on random
    input (converging path chosen) but long runs of symbol 0 keep every route apart.  Wide
    chunks are resolved from their entering sets; the rest stays parallel."""
    Q, A = 64, 4
    rng = np.random.default_rng(64)
    t = np.empty((Q, A), dtype=np.uint16)
    t[:, 0] = (np.arange(Q) + 1) % Q
    t[:, 1:] = rng.integers(0, Q, (Q, 3))
    acc = rng.random(Q) < 0.2
    n = 1 << 21
    x = rng.integers(1, 4, n).astype(np.uint8)
    for start in rng.integers(0, n - 200_000, 6):
        x[start:start + int(rng.integers(10_000, 200_000))] = 0
    with parem.Dfa(t, 3, acc) as d:
        assert d.plan(n)["kernel"] == 3
    for L in (0, 4096, 20_000):
        check(parem, torch_mod, t, 3, acc, x, parem.options(chunk_len=L, kernel="conv"))
    check_find(parem, torch_mod, t, 3, acc, x, parem.options(kernel="conv", chunk_len=4096), cap=5000)
    xz = np.zeros(300_001, np.uint8)   # every chunk wide
    check(parem, torch_mod, t, 3, acc, xz, parem.options(chunk_len=4096, kernel="conv"))


def test_conv_invalid_byte_before_boundaries(parem, torch_mod):
    """Regression: an invalid byte right before a chunk boundary on the converging path (its
    candidate list would be all of Q, larger than the set walk's list) must give ESYMBOL
    with the smallest offset, for every chunk length down to one byte."""
    c = synth.config(3, n=50_000)
    rng = np.random.default_rng(31)
    for L in (1, 2, 3, 16, 1000):
        x = c.make_input().copy()
        bad = np.sort(rng.integers(1, x.size, 3))
        x[bad] = 250
        got = check(parem, torch_mod, c.table, c.start, c.accept, x, parem.options(chunk_len=L, kernel="conv"))
        assert got.status == parem.PAREM_ESYMBOL and got.bad_offset == bad[0]


# ---------------------------------------------------------------- route trace (NEXT-4, Rr)
def test_trace_paper_example_table2(parem, torch_mod):
    """Table II's "Visited states": the routes the join selects are P0 from {0},
    P1 from {1}, P2 from {7} and P3 from {0}; their concatenation is the trace."""
    t = synth.kmp_dfa([0, 1, 2, 1, 4, 4, 3, 4], 5, np.uint32)
    acc = np.zeros(9, dtype=bool)
    acc[8] = True
    x = np.array(["parel".index(ch) for ch in "plaraparallelapareparapl"], np.uint8)
    want = [1, 0, 0, 0, 0, 1,  2, 3, 4, 5, 6, 7,  8, 0, 1, 2, 3, 0,  1, 2, 3, 4, 1, 0]
    with parem.Dfa(t, 0, acc) as d:
        for opts in (parem.options(chunk_len=6, boundary="grid"), None):
            r, st = d.trace(to_dev(torch_mod, x), opts=opts)
            assert r.status == 0 and r.match_count == 1
            assert st.cpu().tolist() == want
        r, st = d.trace(to_dev(torch_mod, x), 5, 14, parem.options(chunk_len=6, boundary="grid"))
        assert st.cpu().tolist() == want[5:14]
        r, st = d.trace(to_dev(torch_mod, x), 7, 7)
        assert st.numel() == 0 and r.match_count == 1
        with pytest.raises(Exception):
            d.trace(to_dev(torch_mod, x), 5, 25)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_trace_configs(parem, torch_mod, k):
    """Every visited state of the CI-sized configs (tiny kernel, converging path) against the
    oracle's prefix walks (oracle.states_at), whole input and an unaligned window."""
    c = synth.config(k, n=(1 << 18) + 5)
    x = c.make_input()
    n = x.size
    ref = oracle.states_at(c.table, c.start, x, np.arange(1, n + 1))
    with parem.Dfa(c.table, c.start, c.accept) as d:
        r, st = d.trace(to_dev(torch_mod, x, offset=3))
        assert r.status == 0
        assert np.array_equal(st.cpu().numpy().astype(np.uint32), ref)
        lo, hi = 70001, 200003
        for opts in (None, parem.options(chunk_len=777, boundary="grid")):
            r, st = d.trace(to_dev(torch_mod, x), lo, hi, opts)
            assert np.array_equal(st.cpu().numpy().astype(np.uint32), ref[lo:hi])


def test_trace_lanes_and_dead(parem, torch_mod):
    """The lanes kernel (partial table: sink state) and death: PAREM_DEAD from the dying symbol on."""
    t = synth.partial_dfa(64, 6, 0.0005, 17, np.uint16)
    acc = np.zeros(64, dtype=bool)
    acc[::5] = True
    x = np.random.default_rng(5).integers(0, 6, 50000).astype(np.uint8)
    ref = oracle.walk(t, 0, acc, x)
    with parem.Dfa(t, 0, acc) as d:
        r, st = d.trace(to_dev(torch_mod, x), opts=parem.options(chunk_len=1000))
    got = st.cpu().numpy().astype(np.uint32)
    # replay the definition on the host (plain walk of the test's own table)
    want = np.empty(x.size, np.uint32)
    s, dead = 0, False
    for i, cc in enumerate(x):
        if not dead:
            nx = int(t[s, cc])
            if nx == 0xFFFF:
                dead = True
            else:
                s = nx
        want[i] = 0xFFFFFFFF if dead else s
    assert np.array_equal(got, want)
    assert (r.final_state == parem.PAREM_DEAD) == dead and r.match_count == ref.match_count
