"""Per-kernel launch counts, mean device time and share of the total from an
`ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv, collections, json, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and r[vi]:
        name = r[ki].split("(")[0].replace("void ", "")
        if "gate_kernel" in name:      # bench.py's timing gate / its probe, not part of a step
            continue
        agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-9))
tot = sum(sum(v) for v in agg.values())
out = {k: {"launches": len(v), "mean_us": 1e6 * sum(v) / len(v), "share": sum(v) / tot}
       for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}
print(json.dumps(out, indent=1))
