"""one input sharded over ranks -- world-size-2 gloo test (CPU) of the
exchange step (one all-gather of the segment maps) and the fold along q0's path
(parem_fold_segment_maps, host C).  The segment maps are built here by the oracle walking
the segment from every candidate of the paper's rule, R = L(last byte of the previous
segment) (reading C1); the folded result must equal the oracle's walk of the whole
input."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_segmap(table, start, accept, seg, prev_symbol):
    """Test-side segment map: for every r in R the oracle's (end, count) over the segment."""
    import oracle
    from paper_1412_1741_b200 import SEGMAP_DTYPE

    Q, A = table.shape
    dead = np.iinfo(table.dtype).max
    m = np.zeros(Q, dtype=SEGMAP_DTYPE)
    if prev_symbol < 0:
        R = [start]
    elif prev_symbol >= A:
        R = list(range(Q))
    else:
        R = sorted({int(v) for v in table[:, prev_symbol] if v != dead})
    status, bad = 0, 0
    for r in R:
        w = oracle.walk(table, r, accept, seg)
        if w.status == oracle.ESYMBOL:
            status, bad = w.status, w.bad_offset
            m[r] = (0, 0, 1)
            continue
        m[r] = (w.match_count, w.final_state, 1)
    return m, status, bad


def cases():
    import synth

    out = []
    c2 = synth.config(2, n=50_001)
    out.append(("kmp", c2.table, c2.start, c2.accept, c2.make_input()))
    c3 = synth.config(3, n=40_000)
    out.append(("random256", c3.table, c3.start, c3.accept, c3.make_input()))
    t = synth.partial_dfa(9, 3, 0.15, 77)          # DEAD entries (reading C9)
    acc = synth.bernoulli(9, 0.3, 77)
    out.append(("partial", t, 0, acc, synth.uniform_symbols(30_000, 3, 78)))
    x = c2.make_input().copy()
    x[31_000] = 9                                   # ESYMBOL in the second segment
    out.append(("esymbol", c2.table, c2.start, c2.accept, x))
    return out


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle
    import paper_1412_1741_b200 as P

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for name, table, start, acc, x in cases():
        n = x.size
        cut = [0, n // 2 + 7, n]                    # uneven split
        seg = x[cut[rank]:cut[rank + 1]]
        prev = int(x[cut[rank] - 1]) if rank > 0 else -1
        m, st, bad = oracle_segmap(table, start, acc, seg, prev)
        got = P.exchange_and_fold(m, st, bad, cut[rank], table.shape[0], start,
                                  np.packbits(np.asarray(acc, bool), bitorder="little"))
        ref = oracle.walk(table, start, acc, x)
        res.append((name, (got.final_state, got.accepted, got.match_count, got.status, got.bad_offset),
                    (ref.final_state, ref.accepted, ref.match_count, ref.status, ref.bad_offset)))
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_fold():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        for name, got, ref in out[rank]:
            if ref[3] != 0:                        # ESYMBOL: status and offset are specified
                assert got[3:] == ref[3:], (rank, name, got, ref)
            else:
                assert got == ref, (rank, name, got, ref)


def test_fold_rejects_unsound_map():
    """A path entering a non-candidate state is an internal error, never a wrong answer."""
    from paper_1412_1741_b200 import SEGMAP_DTYPE, fold_segment_maps, ParemError

    maps = np.zeros((2, 3), dtype=SEGMAP_DTYPE)
    maps[0, 0] = (1, 2, 1)          # q0 = 0 -> 2
    maps[1, 1] = (0, 0, 1)          # segment 1 only admits state 1
    with pytest.raises(ParemError):
        fold_segment_maps(3, 0, np.array([0], np.uint8), maps, [0, 0], [0, 0], [0, 5])
