"""cfg2 DFA at several input sizes: planner row length, grid and GB/s (remainder handling)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1412_1741_b200 as P
c = synth.config(2)
for n in [int(a) for a in sys.argv[1:]] or [1 << 30, 1048576000, 1000000007]:
    x = torch.from_numpy(c.make_input(n)).cuda()
    with P.Dfa(c.table, c.start, c.accept) as d:
        o = P.options(ws_clean=True)
        ws = torch.zeros(d.workspace_bytes(n, o), dtype=torch.uint8, device="cuda")
        res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            d.match_async(x, ws, res, o)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            d.match_async(x, ws, res, o)
        e.record()
        torch.cuda.synchronize()
        pl = d.plan(n, o)
        print("n", n, "L", pl["chunk_len"], "rem", n - pl["num_chunks"] * pl["chunk_len"], "grid", pl["grid_blocks"],
              "GB/s", round(n * 10 / (s.elapsed_time(e) * 1e6), 1), flush=True)
