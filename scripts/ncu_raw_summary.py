"""Summarise `ncu --page raw --csv` exports (one kernel each) into
profiles/ncu_step_summary.json.  usage: ncu_raw_summary.py KEY=raw.csv ..."""
import csv, json, sys
from pathlib import Path
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
    "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_imma_active_pct",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active": "uniform_pipe_pct",
}
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
out_path = Path("profiles/ncu_step_summary.json")
out = json.loads(out_path.read_text()) if out_path.exists() else {}
for arg in sys.argv[1:]:
    key, f = arg.split("=", 1)
    rows = list(csv.reader(open(f)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    rec = {"kernel": vals[hdr.index("Kernel Name")]}
    for m, name in want.items():
        if m in hdr:
            i = hdr.index(m)
            try:
                rec[name] = float(vals[i].replace(",", "")) * scale.get(units[i], 1)
            except ValueError:
                pass
    if "dram_read" in rec and "dram_write" in rec:
        rec["dram_bytes_per_launch"] = rec["dram_read"] + rec["dram_write"]
    out[key] = rec
    print(key, json.dumps(rec))
out_path.write_text(json.dumps(out, indent=1))
