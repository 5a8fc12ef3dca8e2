"""Run parem_find_async on a BASELINE config a few times (profiling helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1412_1741_b200 as P
import synth
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = synth.config(k)
x = torch.from_numpy(c.make_input()).cuda()
with P.Dfa(c.table, c.start, c.accept) as d:
    for _ in range(3):
        r, pos = d.find(x, max_positions=1 << 20)
    torch.cuda.synchronize()
    print(r)
