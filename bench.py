#!/usr/bin/env python
"""bench.py -- input GB/s of PaREM DFA matching on B200 (BASELINE.json metric).

One "step" = one pass of the whole hot path (boundaries + R_i, multi-start chunk
simulation, map composition, result) over one input of a workload, through the C ABI
(parem_match_async) with the input already resident in HBM.

Default run (no flags): ALL five BASELINE.json configs are measured, each for K timed
steps after W warm-up steps, and reported under "per_config"; the line's headline
("value", "roofline", "e2e", "cpu_baseline", ...) is cfg5 -- the largest configuration
(4 GiB input; the 1024-state dense DFA whose 512 KiB table cannot live in one SM's shared
memory: the paper's "large finite automatons").  `--config k` measures config k only
(and makes it the headline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config all|1..5] [--impl ours|reference]

Roofline: every config reports the WHOLE STEP against
  bound = min(HBM copy bandwidth, G_level x 1 byte per lookup)
where G_level is the in-run dependent-gather rate of the memory level holding the table
(shared memory for tables <= 160 KiB, L1/L2 otherwise; merged routes cost ~1 lookup per
input byte), so frac = (n / step time) / bound; the paper-literal lanes kernel is bounded by
G_level / W_exec (route-steps per byte).  The dominant kernel's own rate and share are
reported beside it.

Multi-GPU (torchrun, one process per GPU): every rank matches its own independent input
of the same config (weak scaling, no data-path collective -- the path partitions into
independent problems); value = total bytes of all ranks / max-over-ranks device time.
`--impl reference` times the oracle (single-threaded CPU walk, oracle/) on a bounded
sample of the same workload: the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input GB/s of DFA matching on 1 B200 (device-timed) and % of HBM/lookup roofline"
UNIT = "GB/s"
HEADLINE = 5
L2_BYTES = 126 << 20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, 1965.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_info():
    model, phys = None, set()
    try:
        cur = {}
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ":" not in ln:
                    if cur:
                        phys.add((cur.get("physical id"), cur.get("core id")))
                    cur = {}
                    continue
                k, v = [s.strip() for s in ln.split(":", 1)]
                cur[k] = v
                if k == "model name" and model is None:
                    model = v
            if cur:
                phys.add((cur.get("physical id"), cur.get("core id")))
    except Exception:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(),
            "physical_cores": len(phys) if phys and None not in next(iter(phys)) else None}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)   # first sample lands before the timed region starts
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_input(cfg, rank: int, n: int | None = None):
    """Rank-distinct input of the configured workload (weak scaling): rank 0 gets the
    config's own input; rank r > 0 continues the counter-based stream at offset r*n
    (uniform configs) or uses seed + 1000 r (Markov config)."""
    import synth

    n = cfg.n if n is None else n
    if rank == 0:
        return cfg.make_input(n)
    if cfg.input_kind == "markov":
        return synth.markov_bytes(n, cfg.input_seed + 1000 * rank)
    return synth.uniform_symbols(n, cfg.A, cfg.input_seed, 0, rank * n)


def reduce_max(value: float, dist, device) -> float:
    """Max over ranks (device time of the slowest rank) -- identity when not distributed."""
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def symbol_entropy(x) -> float:
    import numpy as np

    h = np.bincount(x[: min(x.size, 256 << 20)], minlength=256).astype(np.float64)
    p = h[h > 0] / h.sum()
    return float(-(p * np.log2(p)).sum())


def cpu_baseline(cfg, x, budget_s: float = 6.0, max_bytes: int = 256 << 20):
    """The oracle as it stands: single-threaded C walk, pinned to one core, on a bounded
    sample of the input (the first bytes; one rep, more while under budget)."""
    import oracle

    core = None
    try:
        old = os.sched_getaffinity(0)
        core = min(old)
        os.sched_setaffinity(0, {core})
    except Exception:
        old = None
    try:
        probe = x[: min(x.size, 4 << 20)]
        t0 = time.perf_counter()
        oracle.walk(cfg.table, cfg.start, cfg.accept, probe)
        rate = probe.size / max(1e-9, time.perf_counter() - t0)
        nb = int(min(x.size, max_bytes, max(1 << 20, rate * budget_s / 2)))
        sample = x[:nb]
        reps, t_total = 0, 0.0
        while reps < 1 or (t_total < budget_s / 2 and reps < 5):
            t0 = time.perf_counter()
            oracle.walk(cfg.table, cfg.start, cfg.accept, sample)
            t_total += time.perf_counter() - t0
            reps += 1
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    gbs = sample.size * reps / t_total / 1e9
    return {"value": round(gbs, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {sample.size} bytes of the cfg{cfg.index} input x {reps} reps "
                      f"({t_total:.1f} s, single thread pinned to core {core})",
            "host": host_info()}


def run_reference(args):
    """--impl reference: the oracle on the box's host cores, K timed steps over bounded samples."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synth

    k = HEADLINE if args.config == "all" else int(args.config)
    cfg = synth.config(k)
    sample_n = min(cfg.n, args.ref_sample)
    x = cfg.make_input(sample_n)
    for _ in range(args.warmup):
        oracle.walk(cfg.table, cfg.start, cfg.accept, x[: min(x.size, 1 << 20)])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.walk(cfg.table, cfg.start, cfg.accept, x)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = x.size * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded, SURVEY §8(d) recipe)",
        "config": {"workload": f"cfg{cfg.index}: {cfg.name}", "sample_bytes": int(x.size)},
        "cpu_baseline": {"value": round(val, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {x.size} bytes of cfg{cfg.index}, {args.steps} steps",
                         "host": host_info()},
        "e2e": {"value": round(val, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def latest_traffic(cfg_index: int, kernel: str):
    """dram bytes per launch of `kernel` from the newest committed ncu --set full summary
    profiles/r*_ncu_full_cfg<k>_<kernel>.json (r01 files without a kernel suffix hold the
    tiny kernel)."""
    import glob

    pats = [f"r*_ncu_full_cfg{cfg_index}_{kernel}.json"]
    if kernel == "tiny":
        pats.append(f"r*_ncu_full_cfg{cfg_index}.json")
    if kernel == "conv_follow":
        pats.append(f"r*_ncu_full_cfg{cfg_index}_follow.json")
    if kernel == "conv_set":
        pats.append(f"r*_ncu_full_cfg{cfg_index}_set.json")
    cands = []
    for p in pats:
        cands += glob.glob(os.path.join(ROOT, "profiles", p))
    cands.sort(key=lambda s: os.path.basename(s)[:3] + s)
    if not cands:
        return None
    try:
        with open(cands[-1]) as f:
            v = json.load(f).get("dram_bytes_per_launch")
        return {"dram_bytes_per_launch": v, "source": os.path.relpath(cands[-1], ROOT)} if v else None
    except Exception:
        return None


class Micro:
    """In-run roofline micro-benchmarks (denominators measured in the same run)."""

    def __init__(self, P, dev, stream):
        self.P, self.dev, self.stream = P, dev, stream
        self.cache = {}

    def _sink(self):
        import torch

        return torch.full((4,), -1, dtype=torch.int32, device=self.dev)   # sink[1] = 0xFFFFFFFF

    def read_stream(self, xd):
        import ctypes as C

        if "read" in self.cache:
            return self.cache["read"]
        n = xd.numel() & ~15
        ms = self.P.lib().parem_bench_read_stream(C.c_void_p(xd.data_ptr()), n, C.c_void_p(self._sink().data_ptr()), 5,
                                                  C.c_void_p(self.stream.cuda_stream))
        self.cache["read"] = round(n / (ms * 1e-3) / 1e9, 1) if ms > 0 else None
        return self.cache["read"]

    def gather(self, where: int, entries: int):
        """lookups/s of dependent random gathers: where 0 = smem random u32, 1 = global u16
        (L1/L2) over `entries`, 2 = smem lane-private (conflict-free)."""
        import ctypes as C

        import numpy as np
        import torch

        key = (where, entries)
        if key in self.cache:
            return self.cache[key]
        rng = np.random.default_rng(0)
        host = rng.integers(0, 1 << 16, entries).astype(np.uint16)
        # the best of three table allocations: the L2 gather rate differed ~10 % between runs
        # (312-361e9/s for 512 KiB; within one process twelve allocations agree to 0.2 %,
        # tools/placement_probe.py, so it is the box, not the placement), and a peak is the
        # best the level sustains
        best, keep = None, []
        for _ in range(3 if where == 1 else 1):
            tab = torch.from_numpy(host).to(self.dev)
            keep.append(tab)
            lk = C.c_uint64()
            ms = self.P.lib().parem_bench_gather(where, C.c_void_p(tab.data_ptr()), entries, 256,
                                                 C.c_void_p(self._sink().data_ptr()), C.byref(lk), 3,
                                                 C.c_void_p(self.stream.cuda_stream))
            torch.cuda.synchronize()
            if ms > 0:
                v = float(f"{lk.value / (ms * 1e-3):.4g}")
                best = v if best is None else max(best, v)
        self.cache[key] = best
        return best

    def summary(self):
        out = {}
        for k, v in self.cache.items():
            if k == "read":
                out["read_stream_gbs"] = v
            else:
                w, e = k
                nm = {0: "smem_random", 1: "global", 2: "smem_lane_private"}[w]
                out[f"gather_{nm}_{e * (2 if w == 1 else 4) // 1024}KiB_lookups_per_s"] = v
        return out


def timed_steps(dfa, opts, xd, wsb, res, stream, steps, dist, dev, profile=True, sampler_gpu=None):
    """K timed steps (barrier + synchronize on both sides, CUDA events on `stream`);
    returns (device ms total, max over ranks), per-kernel records, clocks."""
    import torch

    import paper_1412_1741_b200 as P

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if profile:
        P.profile(True)   # CUDA events around every kernel the library launches, on `stream`
    with ClockSampler(sampler_gpu if sampler_gpu is not None else dev.index or 0) as clk:
        ev0.record(stream)
        for _ in range(steps):
            dfa.match_async(xd, wsb, res, opts, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    recs = []
    if profile:
        P.profile(False)
        recs = P.profile_read()
    if dist:
        dist.barrier()
    t_ms = reduce_max(ev0.elapsed_time(ev1), dist, dev)
    return t_ms, recs, clk.summary()


def kernel_medians(recs):
    per = {}
    for _, name, ms in recs:
        per.setdefault(name, []).append(ms)
    med = {k: statistics.median(v) for k, v in per.items()}
    tot = {k: sum(v) for k, v in per.items()}
    return med, tot


def run_config(k: int, args, dist, rank: int, ws_: int, dev, micro: Micro, headline: bool):
    import numpy as np
    import torch

    import paper_1412_1741_b200 as P
    import synth

    cfg = synth.config(k)
    n = cfg.n
    t_gen = time.perf_counter()
    x = rank_input(cfg, rank)
    t_gen = time.perf_counter() - t_gen
    xd = torch.from_numpy(x).to(dev)
    stream = torch.cuda.current_stream()
    dfa = P.Dfa(cfg.table, cfg.start, cfg.accept)
    # the workspace starts zero-filled and every completed match leaves it so: no per-call
    # header reset, a step is exactly the path's kernel launches
    opts = P.options(chunk_len=args.chunk_len, boundary=args.boundary, candidates=args.candidates, ws_clean=True,
                     kernel=args.kernel, lookback=args.lookback if args.candidates == "lookback" else 0)
    plan = dfa.plan(n, opts)
    info = dfa.info()
    wsb = torch.zeros(dfa.workspace_bytes(n, opts), dtype=torch.uint8, device=dev)
    res = torch.zeros(64, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        dfa.match_async(xd, wsb, res, opts, stream)
    torch.cuda.synchronize()

    t_ms, recs, clocks = timed_steps(dfa, opts, xd, wsb, res, stream, args.steps, dist, dev)
    kmed, ktot = kernel_medians(recs)
    dominant = max(ktot, key=ktot.get)
    r = P.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
    assert r.status == 0, r
    ms_per_step = t_ms / args.steps
    value = n * ws_ * args.steps / (t_ms / 1e3) / 1e9
    W_exec = r.route_steps / n
    W_grid = info["sum_L"] / cfg.A

    # ---- roofline on the whole step ----
    hbm_peak, sm_mhz_max, peak_src = peaks()
    achieved = n / (ms_per_step * 1e-3) / 1e9          # per GPU
    kern = plan["kernel"]
    tab_entries = (1 << (cfg.A - 1).bit_length()) * (1 << (cfg.Q - 1).bit_length())
    smem_tab = kern in (2, 3) and tab_entries * (4 if cfg.table.dtype == np.uint32 else 2) <= 160 * 1024
    if kern == 1:
        bound = {"bound": "hbm", "peak": hbm_peak, "peak_source": peak_src,
                 "units_per_launch": f"{n} input bytes (tiny kernel: input read once, table in registers/smem)"}
    else:
        if smem_tab:
            G = micro.gather(2, 256)
            level = "smem lane-private gathers (in-run parem_bench_gather where=2)"
        else:
            G = micro.gather(1, min(tab_entries, 1 << 22))
            level = f"L1/L2 gathers over a {min(tab_entries, 1 << 22) * 2 // 1024} KiB table (in-run parem_bench_gather where=1)"
        per_byte = 1.0 if kern == 3 else max(W_exec, 1e-9)
        g_gbs = (G or 0) / per_byte / 1e9
        if g_gbs and g_gbs < hbm_peak:
            bound = {"bound": "smem_lookup" if smem_tab else "l2_lookup", "peak": round(g_gbs, 1),
                     "peak_source": f"{level}: {G:.4g} lookups/s x 1 byte per {per_byte:.4g} lookups"}
        else:
            bound = {"bound": "hbm", "peak": hbm_peak,
                     "peak_source": f"{peak_src}; lookup bound {g_gbs:.0f} GB/s ({level}) is above it"}
        bound["units_per_launch"] = (f"{n} input bytes; converging path: ~1 dependent lookup per byte after routes merge"
                                     if kern == 3 else f"{n} input bytes = {r.route_steps} route-steps")
    bound.update({"unit": UNIT, "achieved": round(achieved, 1), "frac": round(achieved / bound["peak"], 4),
                  "scope": "whole step (all kernels of one match)", "step_ms": round(ms_per_step, 4),
                  "kernel": dominant, "kernel_ms": round(kmed[dominant], 4),
                  "kernel_share": round(ktot[dominant] / max(1e-9, sum(ktot.values())), 3),
                  "kernel_achieved": round(n / (kmed[dominant] * 1e-3) / 1e9, 1),
                  "traffic": latest_traffic(cfg.index, dominant)})
    if bound["traffic"]:
        bound["traffic"]["vs_algorithmic"] = round(bound["traffic"]["dram_bytes_per_launch"] / n, 3)
    if kern == 3 and r.lookups and G:
        # What the converging path executed (parem_result.lookups_k: the set walk's deduplicated
        # sets, the follow's live routes, the join's head walks) against the same gather peak:
        # the fraction of the level's lookup rate the kernels sustain over the whole step.  The
        # gap between this and `frac` is the method's speculation work (lookups per byte > 1).
        lrate = r.lookups / (ms_per_step * 1e-3)
        bound["executed_lookups"] = {
            "lookups_per_launch": r.lookups, "per_input_byte": round(r.lookups / n, 4),
            "rate_per_s": float(f"{lrate:.4g}"), "peak_per_s": float(f"{G:.4g}"),
            "frac_of_gather_peak": round(lrate / G, 4),
            "note": "lookups at distinct states counted by the kernels; SURVEY 8(d) def. 4: achieved lookups/s / G_level"}

    entry = {
        "workload": f"cfg{cfg.index}: {cfg.name}", "n_bytes": n, "states": cfg.Q, "alphabet": cfg.A,
        "value": round(value, 2), "unit": UNIT, "ms_per_step": round(ms_per_step, 4), "steps": args.steps,
        "kernel": {1: "tiny", 2: "lanes", 3: "conv"}.get(kern, kern), "chunks": plan["num_chunks"],
        "chunk_len": plan["chunk_len"],
        "boundary": {0: "grid", 1: "snap"}.get(plan["boundary_policy"], args.boundary),
        "candidates": args.candidates + (f" k={args.lookback}" if args.candidates == "lookback" else ""),
        "roofline": bound, "kernels_ms": {kk: round(v, 4) for kk, v in kmed.items()},
        "W_grid": round(W_grid, 4), "W_exec": round(W_exec, 4),
        "effective_route_steps_per_s": float(f"{r.route_steps / (ms_per_step * 1e-3):.4g}"),
        "result": {"final_state": r.final_state, "accepted": r.accepted, "match_count": r.match_count,
                   "routes": r.routes},
        "gpu_launches": len(recs), "clocks": clocks,
        "l2": "input larger than L2 (no flush needed)" if n > 2 * L2_BYTES else "see single_call / graph_batched",
        "input_gen_s": round(t_gen, 2),
    }
    if cfg.input_kind == "markov":
        entry["symbol_entropy_bits"] = round(symbol_entropy(x), 4)

    # ---- e2e: the same metric through parem_match_host (pinned host buffer, H2D + D2H inside)
    if not args.no_e2e:
        hx = torch.from_numpy(x).pin_memory()
        dfa.match_host(hx)
        torch.cuda.synchronize()
        e_steps = 2 if n > (1 << 30) else 3
        t0 = time.perf_counter()
        for _ in range(e_steps):
            rh = dfa.match_host(hx)
        t_e2e = reduce_max((time.perf_counter() - t0) / e_steps, dist, dev)
        assert (rh.final_state, rh.match_count) == (r.final_state, r.match_count)
        entry["e2e"] = {"value": round(n * ws_ / t_e2e / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(n),
                        "d2h_bytes_per_step": 56, "ms_per_step": round(1e3 * t_e2e, 3), "api": "parem_match_host",
                        "timing": "host wall clock around the synchronous call (H2D from pinned memory inside)"}
        del hx

    # ---- small inputs (cfg1): single call warm and cold (L2 flushed), and the steady-state
    # throughput of a CUDA graph of K matches over K distinct buffers (K n >= 2x L2, so it is
    # HBM-honest; SURVEY §8(d) note 1)
    if n <= (16 << 20):
        flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        warm, cold = [], []
        for i in range(10):
            dfa.match_async(xd, wsb, res, opts, stream)
            e0.record(stream)
            dfa.match_async(xd, wsb, res, opts, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            warm.append(e0.elapsed_time(e1))
            flush.fill_(i)
            e0.record(stream)
            dfa.match_async(xd, wsb, res, opts, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            cold.append(e0.elapsed_time(e1))
        del flush
        entry["single_call"] = {"warm_us": round(1e3 * statistics.median(warm), 2),
                                "cold_us": round(1e3 * statistics.median(cold), 2),
                                "warm_gbs": round(n / (statistics.median(warm) * 1e-3) / 1e9, 2),
                                "cold_gbs": round(n / (statistics.median(cold) * 1e-3) / 1e9, 2),
                                "note": "one match per launch sequence, CUDA events; cold = after writing 2x L2"}
        if not args.no_graph:
            K = max(8, (4 * L2_BYTES + 4 * n) // n)   # K n >= 4x L2 (SURVEY §8(d) note 1): HBM-honest
            bufs = torch.empty((K, n), dtype=torch.uint8, device=dev)
            for i in range(K):
                bufs[i].copy_(torch.from_numpy(rank_input(cfg, rank * K + i)))
            gs = torch.cuda.Stream(device=dev)
            gs.wait_stream(stream)
            with torch.cuda.stream(gs):
                dfa.match_async(bufs[0], wsb, res, opts, gs)
                gs.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=gs):
                    for i in range(K):
                        dfa.match_async(bufs[i], wsb, res, opts, gs)
                graph.replay()
                gs.synchronize()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(gs)
                for _ in range(3):
                    graph.replay()
                g1.record(gs)
                gs.synchronize()
            gms = reduce_max(g0.elapsed_time(g1) / 3, dist, dev)
            entry["graph_batched"] = {"value": round(K * n * ws_ / (gms * 1e-3) / 1e9, 2), "unit": UNIT, "buffers": K,
                                      "bytes_per_buffer": n, "ms_per_graph": round(gms, 4),
                                      "us_per_match": round(1e3 * gms / K, 3),
                                      "note": "CUDA graph of K serialised matches over K distinct buffers"}
            del graph
            # the batched entry (parem_match_batch_async): all K inputs in ONE launch -- the
            # number compared with the 50 % bar for small inputs (SURVEY §8(d) note 1)
            bws = torch.zeros(dfa.batch_workspace_bytes(n, K, opts), dtype=torch.uint8, device=dev)
            bres = torch.zeros(56 * K, dtype=torch.uint8, device=dev)
            for _ in range(3):
                dfa.match_batch_async(bufs, bws, bres, opts, stream)
            torch.cuda.synchronize()
            breps = 10
            P.profile(True)
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(breps):
                dfa.match_batch_async(bufs, bws, bres, opts, stream)
            b1.record(stream)
            torch.cuda.synchronize()
            P.profile(False)
            bk = kernel_medians(P.profile_read())[0]
            bms = reduce_max(b0.elapsed_time(b1) / breps, dist, dev)
            bb = bres.cpu().numpy().tobytes()
            last = P.MatchResult.from_bytes(bb[56 * (K - 1): 56 * K])
            ref_last = P.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])   # graph's last match = input K-1
            assert (last.final_state, last.match_count) == (ref_last.final_state, ref_last.match_count)
            bval = K * n * ws_ / (bms * 1e-3) / 1e9
            hbm_peak = peaks()[0]
            entry["batched"] = {"value": round(bval, 1), "unit": UNIT, "inputs": K, "bytes_per_input": n,
                                "ms_per_batch": round(bms, 4), "us_per_match": round(1e3 * bms / K, 3),
                                "launches_per_batch": len(bk) and 1, "kernels_ms": {kk: round(v, 4) for kk, v in bk.items()},
                                "roofline": {"bound": "hbm", "achieved": round(bval / ws_, 1), "peak": hbm_peak,
                                             "frac": round(bval / ws_ / hbm_peak, 4)},
                                "note": "parem_match_batch_async: K independent matches in one launch; "
                                        "the small-input number compared with the 50 % bar"}
            del bufs, bws, bres

    # ---- NEXT-1: the paper's comparison, PaREM vs Enumeration ----
    if not args.no_enum and args.candidates == "parem":
        eo = P.options(chunk_len=args.chunk_len, boundary=args.boundary, candidates="enum", ws_clean=True,
                       kernel=args.kernel)
        ewsb = torch.zeros(dfa.workspace_bytes(n, eo), dtype=torch.uint8, device=dev)
        for _ in range(2):
            dfa.match_async(xd, ewsb, res, eo, stream)
        torch.cuda.synchronize()
        esteps = max(2, min(args.steps, 5))
        et, erecs, _ = timed_steps(dfa, eo, xd, ewsb, res, stream, esteps, dist, dev)
        er = P.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
        assert (er.final_state, er.match_count) == (r.final_state, r.match_count)
        ems = et / esteps
        entry["enum"] = {"ms_per_step": round(ems, 4), "value": round(n / (ems * 1e-3) / 1e9, 2),
                         "W_exec": round(er.route_steps / n, 4), "routes": er.routes,
                         "parem_speedup_over_enum": round(ems / ms_per_step, 3),
                         "kernels_ms": {kk: round(v, 4) for kk, v in kernel_medians(erecs)[0].items()},
                         "paper": "PaREM 2.3x faster than Enum at 48 threads / 1.07e9 chars, 1.04x at 6 threads / "
                                  "6.69e7 (P:480-483)"}
        del ewsb

    # ---- the paper-literal multi-start kernel (every r in R_i walks the whole chunk, Alg. 1
    # lines 16-25) on the configs whose route-steps it can finish in well under a second
    if not args.no_lanes and kern == 3 and smem_tab:
        lo = P.options(candidates="parem", ws_clean=True, kernel="lanes")
        lwsb = torch.zeros(dfa.workspace_bytes(n, lo), dtype=torch.uint8, device=dev)
        dfa.match_async(xd, lwsb, res, lo, stream)
        torch.cuda.synchronize()
        lt, lrecs, _ = timed_steps(dfa, lo, xd, lwsb, res, stream, 2, dist, dev)
        lr = P.MatchResult.from_bytes(res.cpu().numpy().tobytes()[:56])
        assert (lr.final_state, lr.match_count) == (r.final_state, r.match_count)
        lms = lt / 2
        lkm = kernel_medians(lrecs)[0]
        G = micro.gather(2, 256)
        lk_rate = lr.route_steps / (lms * 1e-3)
        entry["lanes_paper_literal"] = {
            "ms_per_step": round(lms, 3), "value": round(n / (lms * 1e-3) / 1e9, 2),
            "route_steps": lr.route_steps, "W_exec": round(lr.route_steps / n, 3),
            "kernels_ms": {kk: round(v, 4) for kk, v in lkm.items()},
            "roofline": {"bound": "smem_lookup", "achieved": float(f"{lk_rate:.4g}"), "peak": G, "unit": "lookups/s",
                         "frac": round(lk_rate / G, 4) if G else None,
                         "peak_source": "in-run smem lane-private gathers (parem_bench_gather where=2)"},
            "merging_gain": round(lms / ms_per_step, 2),
            "note": "kernel=lanes: every candidate walks the whole chunk (no route merging); merging_gain = its "
                    "step time / the converging path's"}
        del lwsb

    # ---- NEXT-4: match positions (parem_find_async) on the same input, a few steps ----
    if not args.no_find:
        fws = torch.zeros(dfa.find_workspace_bytes(n, opts), dtype=torch.uint8, device=dev)
        cap = max(1024, min(n, 1 << 26))
        fpos = torch.empty(cap, dtype=torch.int64, device=dev)
        fres = torch.zeros(64, dtype=torch.uint8, device=dev)
        for _ in range(2):
            dfa.find_async(xd, fws, fpos, fres, opts, stream)
        torch.cuda.synchronize()
        fsteps = 3
        P.profile(True)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(fsteps):
            dfa.find_async(xd, fws, fpos, fres, opts, stream)
        f1.record(stream)
        torch.cuda.synchronize()
        P.profile(False)
        fk = kernel_medians(P.profile_read())[0]
        fms = reduce_max(f0.elapsed_time(f1) / fsteps, dist, dev)
        fr = P.MatchResult.from_bytes(fres.cpu().numpy().tobytes()[:56])
        assert fr.match_count == r.match_count
        entry["find"] = {"value": round(n * ws_ / (fms * 1e-3) / 1e9, 2), "unit": UNIT, "ms_per_step": round(fms, 4),
                         "positions": int(fr.match_count), "written": int(min(cap, fr.match_count)),
                         "kernels_ms": {kk: round(v, 4) for kk, v in fk.items()},
                         "note": "parem_find_async: the match plus every match end offset (NEXT-4)"}
        del fws, fpos

    # ---- §8(e): ONE input sharded over the ranks (strong scaling of a single input): every
    # rank holds n / N bytes, computes its segment map, one all-gather, fold on every rank.
    # Only meaningful under torchrun (N > 1); wall-clock around the synchronous calls.
    if dist is not None and not args.no_shard:
        seg_n = n // ws_
        seg = xd[:seg_n]
        prev = int(x[seg_n - 1]) if rank > 0 else -1   # this rank's input stands in for T's bytes
        P.shard_match(dfa, seg, prev, rank * seg_n)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(3):
            sr = P.shard_match(dfa, seg, prev, rank * seg_n)
        torch.cuda.synchronize()
        dist.barrier()
        t_sh = reduce_max((time.perf_counter() - t0) / 3, dist, dev)
        entry["sharded"] = {"value": round(seg_n * ws_ / t_sh / 1e9, 2), "unit": UNIT, "ms_per_step": round(1e3 * t_sh, 3),
                            "bytes_per_rank": seg_n, "status": sr.status,
                            "note": "one input of N x bytes_per_rank split over the ranks: parem_segment_map + one "
                                    "all-gather of the maps + fold (SURVEY §8(e)); host wall clock, max over ranks"}
    if not args.no_cpu_baseline and rank == 0 and ws_ == 1:
        entry["cpu_baseline"] = cpu_baseline(cfg, x)
    if args.verify and rank == 0:
        import oracle

        ref = oracle.walk(cfg.table, cfg.start, cfg.accept, x)
        entry["verified"] = (ref.final_state, ref.accepted, ref.match_count) == (r.final_state, r.accepted,
                                                                                  r.match_count)
    if not args.no_micro and headline:
        micro.read_stream(xd)
    dfa.close()
    del xd, wsb, x
    torch.cuda.empty_cache()
    return entry


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="all", help="all (default: cfg1..cfg5, headline cfg5) or 1..5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--boundary", default="auto", choices=["auto", "snap", "grid"])
    ap.add_argument("--candidates", default="parem", choices=["parem", "enum", "lookback"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "tiny", "lanes", "conv"])
    ap.add_argument("--lookback", type=int, default=4, help="k for --candidates lookback (NEXT-2 (i))")
    ap.add_argument("--chunk-len", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-micro", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-find", action="store_true")
    ap.add_argument("--no-enum", action="store_true")
    ap.add_argument("--no-lanes", action="store_true")
    ap.add_argument("--no-shard", action="store_true")
    ap.add_argument("--quick", action="store_true", help="main measurement only (no e2e/find/enum/lanes/cpu)")
    ap.add_argument("--ref-sample", type=int, default=64 << 20)
    ap.add_argument("--verify", action="store_true", help="bit-exact check against the oracle (full size)")
    args = ap.parse_args()
    if args.quick:
        args.no_e2e = args.no_find = args.no_enum = args.no_lanes = args.no_cpu_baseline = args.no_graph = True
        args.no_shard = True
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_1412_1741_b200 as P

    ws_, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dist = None
    if ws_ > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    micro = Micro(P, dev, torch.cuda.current_stream())

    ks = [1, 2, 3, 4, 5] if args.config == "all" else [int(args.config)]
    head = HEADLINE if args.config == "all" else ks[0]
    per = {}
    for k in ks:
        per[f"cfg{k}"] = run_config(k, args, dist, rank, ws_, dev, micro, headline=(k == head))
    h = per[f"cfg{head}"]
    line = {
        "metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": ws_, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded, SURVEY §8(d) recipe; no public dataset in the paper)",
        "config": {"workload": h["workload"] + (" (headline: the largest config)" if args.config == "all" else ""),
                   "n_bytes": h["n_bytes"], "states": h["states"], "alphabet": h["alphabet"],
                   "kernel": h["kernel"], "chunks": h["chunks"], "chunk_len": h["chunk_len"],
                   "boundary": h["boundary"], "candidates": h["candidates"], "l2": h["l2"],
                   "parallelism": f"weak x{ws_} (independent inputs per rank)",
                   "configs_measured": list(per.keys())},
        "roofline": h["roofline"],
        "kernels_ms": h["kernels_ms"], "W_grid": h["W_grid"], "W_exec": h["W_exec"], "result": h["result"],
        "gpu_launches": h["gpu_launches"], "clocks": h["clocks"],
    }
    for key in ("e2e", "cpu_baseline", "enum", "find", "symbol_entropy_bits"):
        if key in h:
            line[key] = h[key]
    line["per_config"] = per
    if not args.no_micro:
        line["micro"] = micro.summary()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
