"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu report
(from the mixed cuda,sass source page; needs -lineinfo).
usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
path, hdr, recs = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        f = lambda s: float(s) if s not in ("", "-") else 0.0
        ie = f(r[len(r) - (len(hdr) - hdr.index("Instructions Executed"))])
        ws = f(r[len(r) - (len(hdr) - hdr.index("Warp Stall Sampling (All Samples)"))])
        recs.append((path, int(r[0]), r[1].strip(), ie, ws))
ti = sum(x[3] for x in recs) or 1
ts = sum(x[4] for x in recs) or 1
print(f"{kre}: total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for f, ln, src, ie, ws in sorted(recs, key=lambda x: -(x[3] / ti + x[4] / ts))[:N]:
    print(f"{f}:{ln:5d} {100*ie/ti:5.1f}% inst {100*ws/ts:5.1f}% stall  {src[:90]}")
