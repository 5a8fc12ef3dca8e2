"""Turn an ncu report into the committed evidence under profiles/:
   profiles/<tag>.json (key metrics, stall mix, dram bytes per launch) and
   profiles/<tag>_details.txt (the ncu details page)."""
import csv, io, json, os, subprocess, sys

rep, tag = sys.argv[1], sys.argv[2]
extra = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    def num(k):
        try:
            return float(d[k].replace(",", ""))
        except Exception:
            return None
    def nbytes(k):
        v = num(k)
        return None if v is None else v * SCALE.get(u.get(k, "byte"), 1)
    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    st = {}
    for h in hdr:
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            v = num(h)
            if v:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
    tot = sum(st.values()) or 1
    keep = ["gpu__time_duration.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
            "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"]
    rec = {"kernel": d.get("Kernel Name"), "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_launch": (rd or 0) + (wr or 0),
           "metrics": {k: (d.get(k), u.get(k)) for k in keep if k in d},
           "stall_pct_top": {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]}}
    rec.update(extra)
    out.append(rec)
res = out[0] if len(out) == 1 else {"launches": out, "dram_bytes_per_launch": out[0]["dram_bytes_per_launch"]}
json.dump(res, open(os.path.join(root, "profiles", tag + ".json"), "w"), indent=1)
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
open(os.path.join(root, "profiles", tag + "_details.txt"), "w").write(det)
print(json.dumps(res, indent=1)[:1500])
