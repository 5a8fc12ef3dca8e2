"""Key raw metrics per kernel of an ncu report: python tools/ncu_metrics.py REPORT [regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = {"gpu__time_duration.sum": "ms", "launch__registers_per_thread": "regs", "launch__grid_size": "grid",
        "launch__block_size": "block", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%", "smsp__inst_executed.sum": "inst",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "lds_conf",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "lds_wf", "lts__t_sector_hit_rate.pct": "L2hit%",
        "l1tex__t_sector_hit_rate.pct": "L1hit%", "dram__bytes_read.sum": "dramR", "dram__bytes_write.sum": "dramW",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum": "atom_conf",
        "lts__t_sectors_srcunit_tex_op_read.sum": "L2sectR", "sm__cycles_elapsed.avg.per_second": "clk"}
stallk = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if kre and not kre.search(d.get("Kernel Name", "")):
        continue
    print(d.get("Kernel Name", "")[:90])
    print("  ", {v: d.get(k) for k, v in want.items() if k in d})
    st = {}
    for h in stallk:
        try:
            st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[h].replace(",", ""))
        except Exception:
            pass
    tot = sum(st.values()) or 1
    print("   stalls%", {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:7]})
