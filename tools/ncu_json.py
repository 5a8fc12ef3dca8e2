"""Write the per-launch summary of one kernel from an ncu --set full report as JSON (the file
bench.py reads `traffic` from: profiles/rNN_ncu_full_cfg<k>_<kernel>.json).
usage: python tools/ncu_json.py REPORT KERNEL_REGEX OUT.json [note]"""
import csv, io, json, re, subprocess, sys

rep, kre, out = sys.argv[1], re.compile(sys.argv[2]), sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1, "nsecond": 1e-6,
         "us": 1e-3, "ms": 1, "ns": 1e-6}


def val(d, k):
    i = hdr.index(k)
    return float(d[k].replace(",", "")) * scale.get(units[i], 1)


recs = [dict(zip(hdr, r)) for r in rows[2:] if kre.search(r[hdr.index("Kernel Name")])]
d = recs[-1]
res = {"kernel": d["Kernel Name"], "launches_in_report": len(recs), "gpu_time_ms": val(d, "gpu__time_duration.sum"),
       "dram_bytes_per_launch": val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum"),
       "registers": int(float(d["launch__registers_per_thread"])),
       "achieved_occupancy_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
       "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"])}
for k, nm in (("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_load_bank_conflicts"),
              ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem_load_wavefronts"),
              ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem_store_bank_conflicts"),
              ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem_store_wavefronts"),
              ("lts__t_sector_hit_rate.pct", "l2_hit_pct"), ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct")):
    if k in hdr:
        res[nm] = float(d[k].replace(",", ""))
st = {}
for h in hdr:
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[h].replace(",", ""))
        except ValueError:
            pass
tot = sum(st.values()) or 1
res["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
res["source"] = rep + (" -- " + note if note else "")
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
