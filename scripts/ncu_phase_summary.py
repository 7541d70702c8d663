"""Group an ncu source page of the fused step kernel by phase (marker
comments in step_kernel.cuh).  Usage: ncu_phase_summary.py REPORT|SOURCE.csv [SRC]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_1504_05158_b200/csrc/step_kernel.cuh"
lines = open(src).read().split("\n")
markers = [("setup", "// ---- per-column registers"),
           ("velocity", "// ================= phase 1: velocity"),
           ("stats", "// ================= normalisation"),
           ("agg:init", "// ================= phase 2: aggregation"),
           ("agg:endgame", "// ---- endgame"),
           ("agg:bulk", "// ---- bulk step"),
           ("agg:round", "// ---- one round"),
           ("agg:ties", "// ---- ties"),
           ("agg:retire", "// ---- retire row"),
           ("agg:rescans", "// ---- cooperative rescans"),
           ("agg:end", "// the tile is no longer read"),
           ("goal", "// ================= phase 3: goal"),
           ("pbest", "// ================= phase 4a"),
           ]
bounds = []
kstart = next(i for i, l in enumerate(lines) if l.startswith("step_kernel(const")) + 1
for name, m in markers:
    idx = next((i for i, l in enumerate(lines) if m in l), None)
    if idx is not None:
        bounds.append((idx + 1, name))
bounds.sort()


def region(fname, ln):
    if fname != src.split("/")[-1]:
        return fname
    if ln < kstart:
        return "helpers (rare paths, keys)"
    name = "kernel:prologue"
    for b, nm in bounds:
        if ln >= b:
            name = nm
    return name


if rep.endswith(".csv"):      # an exported source page (--print-source cuda,sass)
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
ins = defaultdict(int)
smp = defaultdict(int)
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    try:
        i = int(r[hdr.index("Instructions Executed")] or 0)
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ln = int(r[0])
    except ValueError:
        continue
    g = region(fname, ln)
    ins[g] += i
    smp[g] += s
ti, ts = sum(ins.values()), sum(smp.values())
print(f"total warp-instructions {ti:,}  stall samples {ts:,}")
for g in sorted(ins, key=lambda g: -smp[g]):
    print(f"{100 * ins[g] / ti:6.1f}% inst {100 * smp[g] / ts:6.1f}% samp  {g}")
