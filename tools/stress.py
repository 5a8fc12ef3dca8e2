"""Randomised stress of every path against the oracle (ad hoc; many seeds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth, paper_1412_1741_b200 as P

bad = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 300):
    rng = np.random.default_rng(int(os.environ.get("STRESS_BASE", "100000")) + seed)
    Q = int(rng.choice([1, 2, 4, 9, 17, 32, 33, 64, 200, 700, 3000]))
    A = int(rng.choice([1, 2, 3, 4, 6, 26, 255, 256]))
    partial = rng.random() < 0.3
    dt = np.uint16 if rng.random() < 0.6 else np.uint32
    t = synth.partial_dfa(Q, A, float(rng.choice([0.01, 0.2])), seed, dt) if partial else synth.random_dfa(Q, A, seed, dt)
    acc = rng.random(Q) < float(rng.choice([0.0, 0.1, 0.6, 1.0]))
    q0 = int(rng.integers(0, Q))
    n = int(rng.choice([0, 1, 5, 64, 1000, 33333, 200001, 1 << 20]))
    kind = rng.choice(["uniform", "runs", "zeros", "bad"])
    x = rng.integers(0, A, n).astype(np.uint8)
    if kind == "runs" and n:
        x = np.repeat(rng.integers(0, A, n // 100 + 1).astype(np.uint8), 100)[:n]
    elif kind == "zeros":
        x = np.zeros(n, np.uint8)
    elif kind == "bad" and n and A < 256:
        x[rng.integers(0, n, 2)] = 255
    opts = P.options(chunk_len=int(rng.choice([0, 0, 1, 7, 64, 500, 4096])),
                     boundary=str(rng.choice(["auto", "grid", "snap"])),
                     candidates=str(rng.choice(["parem", "parem", "enum"])))
    # the converging path's opt-in variants (read by the planner on every call)
    os.environ["PAREM_CONV_TMA"] = str(int(rng.random() < 0.3))
    os.environ["PAREM_CONV_REP"] = str(int(rng.choice([0, 8, 16, 116, 116])))   # 116: byte-entry table (the default where it applies)
    os.environ["PAREM_CONV_HYB"] = str(int(rng.random() < 0.3))   # hybrid follow table (Q <= 1024, L2 tables)
    os.environ["PAREM_CONV_CPT"] = str(int(rng.choice([1, 1, 2])))  # chunks per follow thread (interleaved walk)
    ref = oracle.walk(t, q0, acc, x)
    buf = torch.empty(n + 32, dtype=torch.uint8, device="cuda")
    off = int(rng.integers(0, 16))
    xd = buf[off:off + n]
    if n:
        xd.copy_(torch.from_numpy(x))
    try:
        with P.Dfa(t, q0, acc) as d:
            r = d.match(xd, opts)
            rf, pos = d.find(xd, max_positions=100, opts=opts)
            # one input sharded into 1..3 segments: segment maps + fold
            G = int(rng.integers(1, 4))
            cuts = sorted([0, n] + [int(v) for v in rng.integers(0, n + 1, G - 1)])
            maps, sts, bads = [], [], []
            for g in range(G):
                seg = xd[cuts[g]:cuts[g + 1]]
                m, st_, b_ = d.segment_map(seg, int(x[cuts[g] - 1]) if cuts[g] > 0 else -1)
                maps.append(m); sts.append(st_); bads.append(b_)
            rs = P.fold_segment_maps(Q, q0, d.accept_bitmap, np.stack(maps), sts, bads, cuts[:-1])
            # the same input twice more as a batch of independent inputs
            rb = d.match_batch(torch.stack([xd, xd, xd]) if n else xd.reshape(0, 0)) if n else []
        if ref.status == oracle.ESYMBOL:
            ok = r.status == P.PAREM_ESYMBOL and r.bad_offset == ref.bad_offset
            ok = ok and rs.status == P.PAREM_ESYMBOL and rs.bad_offset == ref.bad_offset
            ok = ok and all(b.status == P.PAREM_ESYMBOL and b.bad_offset == ref.bad_offset for b in rb)
        else:
            pr, cnt = oracle.positions(t, q0, acc, x, cap=100)
            want = (ref.final_state, ref.accepted, ref.match_count)
            ok = (r.status == 0 and (r.final_state, r.accepted, r.match_count) == want
                  and rf.match_count == cnt and pos.cpu().numpy().astype(np.uint64).tolist() == pr.tolist())
            ok = ok and rs.status == 0 and (rs.final_state, rs.accepted, rs.match_count) == want
            ok = ok and all(b.status == 0 and (b.final_state, b.accepted, b.match_count) == want for b in rb)
    except Exception as e:
        ok = False
        print("EXC", e)
    if not ok:
        bad += 1
        print("MISMATCH seed", seed, Q, A, partial, n, kind, opts.chunk_len, opts.boundary_policy, opts.candidates, r if 'r' in dir() else None, ref, flush=True)
print("stress done, mismatches:", bad)
