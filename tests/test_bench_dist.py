"""World-size-2 gloo test of bench.py's multi-rank logic (CPU): rank-distinct inputs
(weak scaling, no data-path collective) and the max-over-ranks device time."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import bench
    import synth

    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.config(2, n=4096)
    x = bench.rank_input(cfg, rank)
    t = bench.reduce_max(1.5 + rank, dist, torch.device("cpu"))
    digest = int(np.frombuffer(x.tobytes(), dtype=np.uint64).sum(dtype=np.uint64))
    q.put((rank, t, digest, bool((x == cfg.make_input()).all())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_weak_scaling_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, d0, same0), (r1, t1, d1, same1) = res
    assert t0 == t1 == 2.5            # max over ranks, seen by every rank
    assert same0 and not same1        # rank 0 = the config's input, rank 1 distinct
    assert d0 != d1
