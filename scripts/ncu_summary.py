"""Summarise an `ncu --set full` report of the fused step kernel into
profiles/ncu_step_summary.json (per-launch DRAM traffic etc.) and print it.

usage: ncu_summary.py REPORT KEY [--out profiles/ncu_step_summary.json]"""
import csv, io, json, subprocess, sys
from pathlib import Path

rep, key = sys.argv[1], sys.argv[2]
out = Path(sys.argv[4] if len(sys.argv) > 4 else "profiles/ncu_step_summary.json")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = {
    "gpu__time_duration.sum": "duration_s",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__pcsamp_sample_count": "stall_samples",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
rec = {}
for r in vals:
    name = r[hdr.index("Kernel Name")]
    if "step_kernel" not in name:
        continue
    d = {"kernel": name}
    for m, k in want.items():
        if m in hdr:
            i = hdr.index(m)
            v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else None
            u = units[i]
            if v is not None and u in scale:
                v *= scale[u]
            d[k] = v
    d["dram_bytes_per_launch"] = (d.get("dram_read") or 0) + (d.get("dram_write") or 0)
    rec = d
    break
db = json.loads(out.read_text()) if out.exists() else {}
db[key] = rec
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps(db, indent=1))
print(json.dumps(rec, indent=1))
