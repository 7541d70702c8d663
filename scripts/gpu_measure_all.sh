# Round measurements: bench lines of every BASELINE config, the reference arm,
# launch lists and ncu summaries (reports stay in /tmp on the box; only the
# summaries and CSV exports come back, under gpurun_out/m).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/m
rm -f gpurun_out/m/*
timeout 900 python bench.py > gpurun_out/m/bench_config3.json 2> gpurun_out/m/err.log; echo "config3 rc=$?" >> gpurun_out/m/err.log
timeout 600 python bench.py --impl reference > gpurun_out/m/bench_reference.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config1 --no-cpu --steps 400 --graph > gpurun_out/m/bench_config1.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config2 --no-cpu --steps 200 > gpurun_out/m/bench_config2.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --no-cpu --steps 200 > gpurun_out/m/bench_config4.json 2>> gpurun_out/m/err.log
timeout 600 python bench.py --preset config5 --no-cpu --steps 30 --warmup 3 > gpurun_out/m/bench_config5.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --precision fp64 --no-cpu --steps 200 > gpurun_out/m/bench_config3_fp64.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n50.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n100_10k.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config5 --velocity-only --no-cpu --steps 20 --warmup 3 > gpurun_out/m/bench_velocity_n256_2k.json 2>> gpurun_out/m/err.log
# launch lists (the kernel's share of the step)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > /tmp/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches_c2.csv python bench.py --preset config2 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > /tmp/l2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches_c5.csv python bench.py --preset config5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > /tmp/l5.log 2>&1
# full captures: fused step (early launch and a late one), velocity-only, 2-opt kernels
prof() {  # name kernel-regex skip bench-args...
  name=$1; k=$2; skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$name python bench.py --no-cpu --e2e-steps 0 "$@" > /tmp/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/m/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/m/${name}_details.txt 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/m/${name}_source.csv 2>/dev/null
}
prof prof_step step_kernel 10 --steps 8 --warmup 5
prof prof_step_late step_kernel 300 --steps 300 --warmup 5
prof prof_vel50 step_kernel 3 --velocity-only --steps 3 --warmup 2
prof prof_twoopt_c5 twoopt_tc 2 --preset config5 --steps 3 --warmup 3
prof prof_twoopt_c2 twoopt_tc 2 --preset config2 --steps 3 --warmup 3
python scripts/ncu_phase_summary.py /tmp/prof_step.ncu-rep > gpurun_out/m/ncu_step_phases.txt 2>&1
python scripts/ncu_phase_summary.py /tmp/prof_step_late.ncu-rep > gpurun_out/m/ncu_step_late_phases.txt 2>&1
bash scripts/gpu_velocity_sweep.sh > gpurun_out/m/velocity_sweep.log 2>&1
cp gpurun_out/vs/sweep.json gpurun_out/m/velocity_sweep.json 2>/dev/null
for f in gpurun_out/m/bench_*.json; do echo "$f: $(python -c "
import json,sys
d=json.load(open('$f')); r=d.get('roofline') or {}
print(round(d['value']), 'ms', round(d.get('ms_per_step',0),4), 'kern', r.get('kernel_ms'), 'frac', r.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'))")"; done
tail -3 gpurun_out/m/err.log
du -sh gpurun_out
