"""Per-address-bucket instruction counts and no-instruction stall samples
from an ncu SASS source page (--print-source sass --csv).  Shows where the
instruction-fetch stalls land and how much code is actually executed.
usage: sass_noinst.py page.csv [bucket_bytes]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
h = rows[1]
ia, ii, ins = h.index("Address"), h.index("Instructions Executed"), h.index("stall_no_inst")
iall = h.index("Warp Stall Sampling (All Samples)")
base = None
agg = {}
exec_bytes = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    a = int(r[ia], 16)
    if base is None:
        base = a
    off = a - base
    b = off // bucket
    e = agg.setdefault(b, [0, 0, 0, 0])
    n = int(r[ii] or 0)
    e[0] += n; e[1] += int(r[ins] or 0); e[2] += int(r[iall] or 0)
    if n:
        e[3] += 1; exec_bytes += 16
tot_i = sum(v[0] for v in agg.values()); tot_n = sum(v[1] for v in agg.values()); tot_s = sum(v[2] for v in agg.values())
print(f"code {16*(len(rows)-2)} B, executed {exec_bytes} B; inst {tot_i}, no_inst samples {tot_n} of {tot_s}")
for b in sorted(agg):
    i, n, s, x = agg[b]
    if i or n:
        print(f"{b*bucket:7d} inst {100*i/tot_i:5.1f}%  noinst {100*n/max(tot_n,1):5.1f}%  samp {100*s/tot_s:5.1f}%  exec_instrs {x}")
