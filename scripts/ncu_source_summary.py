"""Summarise an ncu source page (cuda view) by source line: instructions
executed and stall samples.  Usage: ncu_source_summary.py report.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if r[2] != "-":
        continue   # SASS rows; keep the per-source-line aggregates
    try:
        ins = int(r[hdr.index("Instructions Executed")] or 0)
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    rows.append((ins, samp, fname, r[0], r[1].strip()[:90]))
tot_i = sum(r[0] for r in rows) or 1
tot_s = sum(r[1] for r in rows) or 1
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for ins, samp, f, ln, src in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{100*ins/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% samp  {f}:{ln}  {src}")
