import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth, paper_1412_1741_b200 as P
seed = 125
rng = np.random.default_rng(100000 + seed)
Q = int(rng.choice([1, 2, 4, 9, 17, 32, 33, 64, 200, 700, 3000])); A = int(rng.choice([1, 2, 3, 4, 6, 26, 255, 256]))
partial = rng.random() < 0.3; dt = np.uint16 if rng.random() < 0.6 else np.uint32
t = synth.partial_dfa(Q, A, float(rng.choice([0.01, 0.2])), seed, dt) if partial else synth.random_dfa(Q, A, seed, dt)
acc = rng.random(Q) < float(rng.choice([0.0, 0.1, 0.6, 1.0])); q0 = int(rng.integers(0, Q))
n = int(rng.choice([0, 1, 5, 64, 1000, 33333, 200001, 1 << 20])); kind = rng.choice(["uniform", "runs", "zeros", "bad"])
x = rng.integers(0, A, n).astype(np.uint8)
if kind == "bad": x[rng.integers(0, n, 2)] = 255
L = int(rng.choice([0, 0, 1, 7, 64, 500, 4096])); b = str(rng.choice(["auto", "grid", "snap"])); c = str(rng.choice(["parem", "parem", "enum"]))
print(Q, A, partial, dt, n, kind, L, b, c, flush=True)
which = sys.argv[1]
xd = torch.from_numpy(x).cuda()
with P.Dfa(t, q0, acc) as d:
    o = P.options(chunk_len=int(sys.argv[2]) if len(sys.argv) > 2 else L, boundary=b, candidates=c, kernel=which)
    print(d.plan(n, o), flush=True)
    r = d.match(xd, o)
    print(r, oracle.walk(t, q0, acc, x), flush=True)
