# velocity/normalise phase (velocity-only build of the fused kernel) across n and P -> gpurun_out/vs/sweep.json
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/vs
rm -f gpurun_out/vs/*.json
run() {  # tag args...
  tag=$1; shift
  timeout 300 python bench.py --velocity-only --no-cpu --steps 50 --warmup 5 "$@" > gpurun_out/vs/$tag.json 2>> gpurun_out/vs/err.log
}
run n12_P100 --preset config1
run n30_P10k --preset config2
run n50_P80k --preset config3
run n100_P10k --preset config4
run n256_P2k --preset config5
for s in 20 50 200 500; do run n100_P${s}00 --n 100 --swarms $s; done
for s in 100 200 400 1600; do run n50_P${s}00 --n 50 --swarms $s; done
python - <<'PY'
import json, glob, os
out = {}
for f in sorted(glob.glob("gpurun_out/vs/n*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        out[os.path.basename(f)[:-5]] = {"error": str(e)}; continue
    r = d["roofline"]
    out[os.path.basename(f)[:-5]] = {"n": d["config"]["n"], "particles": d["config"]["particles"],
        "kernel_us": round(1000 * r["kernel_ms"], 2), "bytes_per_launch": r["algorithmic_bytes_per_launch"],
        "achieved_gbs": round(r["achieved"], 1), "frac_of_measured_hbm": round(r["frac"], 4),
        "clocks": d.get("clocks")}
json.dump(out, open("gpurun_out/vs/sweep.json", "w"), indent=1)
for k, v in out.items(): print(k, v.get("kernel_us"), v.get("achieved_gbs"), v.get("frac_of_measured_hbm"))
PY
tail -3 gpurun_out/vs/err.log
