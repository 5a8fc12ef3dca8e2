"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth, paper_1412_1741_b200 as P

def run(table, start, acc, x, **kw):
    ref = oracle.walk(table, start, acc, x)
    xd = torch.from_numpy(x).cuda()
    with P.Dfa(table, start, acc) as d:
        r = d.match(xd, P.options(**kw))
        rf, pos = d.find(xd, max_positions=1000, opts=P.options(**kw))
    assert (r.final_state, r.match_count) == (ref.final_state, ref.match_count), (kw, r, ref)
    assert rf.match_count == ref.match_count
    print("ok", kw, r.match_count, flush=True)

for k in (1, 2, 3, 5):
    c = synth.config(k, n=(1 << 18) + 77)
    x = c.make_input()
    run(c.table, c.start, c.accept, x)
c = synth.config(3, n=(1 << 18) + 77)
run(c.table, c.start, c.accept, c.make_input(), kernel="lanes")
run(c.table, c.start, c.accept, c.make_input(), kernel="conv", chunk_len=333)
run(c.table, c.start, c.accept, np.zeros(200001, np.uint8), kernel="conv")
c = synth.config(2, n=(1 << 18) + 77)
run(c.table, c.start, c.accept, c.make_input(), boundary="snap")
run(c.table, c.start, c.accept, c.make_input(), chunk_len=97, candidates="enum")
t = synth.partial_dfa(40, 4, 0.05, 3, np.uint16)
run(t, 0, np.arange(40) % 3 == 0, np.random.default_rng(1).integers(0, 4, 100000).astype(np.uint8))
print("all ok")
