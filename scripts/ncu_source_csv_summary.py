"""Per-source-line instructions and stall samples from an exported
`ncu --page source --csv --print-source cuda,sass` file.  usage: FILE [top]"""
import csv, sys
f = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, hdr, fname = [], None, None
for r in csv.reader(open(f)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    d = dict(zip(hdr, r))
    try:
        rows.append((int(d["Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0),
                     int(d.get("stall_no_inst") or 0), fname, r[0], r[1].strip()[:90]))
    except (ValueError, KeyError):
        pass
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
tn = sum(x[2] for x in rows)
print(f"total warp-instructions {ti:,}  stall samples {ts:,}  (no_instruction {tn:,})")
for ins, samp, ni, fn, ln, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{100*ins/ti:5.1f}% inst {100*samp/ts:5.1f}% samp  {fn}:{ln}  {src}")
