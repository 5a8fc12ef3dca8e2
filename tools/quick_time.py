"""Scratch timing: device-timed matches for selected configs (not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1412_1741_b200 as P

def run(k, n=None, reps=5, **kw):
    c = synth.config(k, n=n)
    t0 = time.time(); x = c.make_input(); tg = time.time() - t0
    xd = torch.from_numpy(x).to("cuda")
    d = P.Dfa(c.table, c.start, c.accept)
    opts = P.options(**kw)
    plan = d.plan(x.size, opts)
    ws = torch.empty(d.workspace_bytes(x.size, opts), dtype=torch.uint8, device="cuda")
    res = torch.zeros(64, dtype=torch.uint8, device="cuda")
    d.match_async(xd, ws, res, opts); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); d.match_async(xd, ws, res, opts); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    r = P.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
    ms = min(ts)
    print(f"cfg{k} n={x.size} {kw} plan(kernel={plan['kernel']} grid={plan['grid_blocks']} thr={plan['block_threads']} p={plan['num_chunks']} L={plan['chunk_len']} slots={plan['slots']}) "
          f"ms={ms:.3f} med={sorted(ts)[len(ts)//2]:.3f} GB/s={x.size/ms/1e6:.1f} W_exec={r.route_steps/x.size:.3f} count={r.match_count} final={r.final_state} st={r.status} gen={tg:.1f}s", flush=True)
    d.close()

if __name__ == "__main__":
    which = [int(a) for a in sys.argv[1:]] or [1, 2, 3]
    for k in which:
        run(k)
        if k == 2:
            run(k, boundary="grid")
