"""GPU parity of batched matching (parem_match_batch_async): every input of a batch is an
independent match from q0 and must equal the oracle's walk of that input alone --
final state, accept flag, match count, status and (input-local) bad offset, bit-exact."""
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


def batch_inputs(cfg, count, n, seed_offset=0):
    return np.stack([synth.uniform_symbols(n, cfg.A, cfg.input_seed + 7, 0, (i + seed_offset) * n)
                     for i in range(count)])


def run_batch(parem, torch, cfg, X, opts=None, reuse=1):
    count, n = X.shape
    with parem.Dfa(cfg.table, cfg.start, cfg.accept) as d:
        xd = torch.from_numpy(X).cuda()
        ws = torch.zeros(d.batch_workspace_bytes(n, count, opts), dtype=torch.uint8, device="cuda")
        res = torch.zeros(56 * count, dtype=torch.uint8, device="cuda")
        out = None
        for _ in range(reuse):   # the workspace stays clean between calls (PAREM_FLAG_WS_CLEAN)
            d.match_batch_async(xd, ws, res, opts)
            b = res.cpu().numpy().tobytes()
            out = [parem.MatchResult.from_bytes(b[56 * i: 56 * (i + 1)]) for i in range(count)]
        return out


def expect_all(cfg, X, got):
    for i in range(X.shape[0]):
        ref = oracle.walk(cfg.table, cfg.start, cfg.accept, X[i])
        g = got[i]
        if ref.status == oracle.ESYMBOL:   # only status and offset are specified (parem.h)
            assert (g.status, g.bad_offset) == (ref.status, ref.bad_offset), (i, g, ref)
            continue
        assert (g.final_state, g.accepted, g.match_count, g.status, g.bad_offset) == \
            (ref.final_state, ref.accepted, ref.match_count, ref.status, ref.bad_offset), (i, g, ref)
        assert g.routes >= 1 and g.num_chunks >= 1


@pytest.mark.parametrize("k,count,n", [(1, 16, 1 << 20), (2, 8, 1 << 16), (1, 3, 1 << 16), (2, 5, 3 << 17)])
def test_batch_single_launch_matches_oracle(parem, torch_mod, k, count, n):
    cfg = synth.config(k)
    X = batch_inputs(cfg, count, n)
    got = run_batch(parem, torch_mod, cfg, X, parem.options(ws_clean=True), reuse=2)
    expect_all(cfg, X, got)


@pytest.mark.parametrize("k,count,n,L", [(1, 5, 1 << 16, 1024), (1, 7, 1 << 16, 256), (2, 9, 1 << 17, 256),
                                         (2, 3, 1 << 15, 512), (1, 33, 1 << 20, 4096), (2, 4, 1 << 20, 1024),
                                         (2, 2, 1 << 21, 64)])
def test_batch_short_inputs_share_tiles(parem, torch_mod, k, count, n, L):
    """Forced chunk lengths: inputs of fewer chunks than a CTA tile (cpi = n / L = 64 .. 512)
    are packed several per tile (one sub-tile map each), a partly filled last tile included;
    cpi >= 1024 keeps whole tiles per input.  Stats are those of a single GRID match."""
    cfg = synth.config(k)
    X = batch_inputs(cfg, count, n, 21)
    got = run_batch(parem, torch_mod, cfg, X, parem.options(ws_clean=True, chunk_len=L), reuse=2)
    expect_all(cfg, X, got)
    assert all(g.num_chunks == n // L for g in got)
    b = oracle.grid_boundaries(n, L)
    for i in (0, count - 1):
        assert (got[i].routes, got[i].route_steps) == oracle.route_stats(cfg.table, X[i], b)


@pytest.mark.parametrize("n", [100003, 1000, 1, 65536 + 16])
def test_batch_fallback_sizes(parem, torch_mod, n):
    # not whole tiles: the inputs are matched one after another (same results)
    cfg = synth.config(2)
    X = batch_inputs(cfg, 4, n, 3)
    expect_all(cfg, X, run_batch(parem, torch_mod, cfg, X))


def test_batch_invalid_byte_is_local(parem, torch_mod):
    cfg = synth.config(2)
    X = batch_inputs(cfg, 6, 1 << 16, 9)
    X[2, 777] = 200           # input 2: ESYMBOL at local offset 777
    X[4, 65535] = 4           # input 4: the very last byte
    got = run_batch(parem, torch_mod, cfg, X)
    expect_all(cfg, X, got)
    assert got[2].status == parem.PAREM_ESYMBOL and got[2].bad_offset == 777
    assert got[4].status == parem.PAREM_ESYMBOL and got[4].bad_offset == 65535
    assert got[3].status == 0


def test_batch_stats_equal_single_matches(parem, torch_mod):
    cfg = synth.config(2)
    X = batch_inputs(cfg, 4, 1 << 17, 5)
    got = run_batch(parem, torch_mod, cfg, X)
    opts = parem.options(chunk_len=got[0].num_chunks and (X.shape[1] // got[0].num_chunks), boundary="grid")
    with parem.Dfa(cfg.table, cfg.start, cfg.accept) as d:
        for i in range(X.shape[0]):
            one = d.match(torch_mod.from_numpy(X[i]).cuda(), opts)
            assert (one.routes, one.route_steps, one.num_chunks) == (got[i].routes, got[i].route_steps,
                                                                     got[i].num_chunks)


def test_batch_graph_capture(parem, torch_mod):
    torch = torch_mod
    cfg = synth.config(1)
    X = batch_inputs(cfg, 8, 1 << 16, 11)
    count, n = X.shape
    with parem.Dfa(cfg.table, cfg.start, cfg.accept) as d:
        xd = torch.from_numpy(X).cuda()
        opts = parem.options(ws_clean=True)
        ws = torch.zeros(d.batch_workspace_bytes(n, count, opts), dtype=torch.uint8, device="cuda")
        res = torch.zeros(56 * count, dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            d.match_batch_async(xd, ws, res, opts, s)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                d.match_batch_async(xd, ws, res, opts, s)
            res.zero_()
            g.replay()
            g.replay()
            s.synchronize()
        b = res.cpu().numpy().tobytes()
        got = [parem.MatchResult.from_bytes(b[56 * i: 56 * (i + 1)]) for i in range(count)]
    expect_all(cfg, X, got)


def test_batch_empty(parem, torch_mod):
    cfg = synth.config(1)
    with parem.Dfa(cfg.table, cfg.start, cfg.accept) as d:
        x = torch_mod.zeros((0, 64), dtype=torch_mod.uint8, device="cuda")
        assert d.match_batch(x) == []
