cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/m
rm -f gpurun_out/m/*.json
timeout 900 python bench.py > gpurun_out/m/bench_config3.json 2> gpurun_out/m/err.log; echo "config3 rc=$?" >> gpurun_out/m/err.log
timeout 600 python bench.py --impl reference > gpurun_out/m/bench_reference.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config1 --no-cpu --steps 400 --graph > gpurun_out/m/bench_config1.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config2 --no-cpu --steps 200 > gpurun_out/m/bench_config2.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --no-cpu --steps 200 > gpurun_out/m/bench_config4.json 2>> gpurun_out/m/err.log
timeout 600 python bench.py --preset config5 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/m/bench_config5.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --precision fp64 --no-cpu --steps 200 > gpurun_out/m/bench_config3_fp64.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n50.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n100_10k.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/m/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/m/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 1 -o gpurun_out/m/prof_step python bench.py --steps 8 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/m/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/m/prof_vel50 python bench.py --velocity-only --steps 3 --warmup 2 --no-cpu > gpurun_out/m/ncu_vel.log 2>&1
for f in gpurun_out/m/*.json; do echo "$f: $(python -c "
import json,sys
d=json.load(open('$f')); r=d.get('roofline') or {}
print(round(d['value']), 'ms', round(d.get('ms_per_step',0),4), 'kern', r.get('kernel_ms'), 'frac', r.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'))")"; done
tail -3 gpurun_out/m/err.log
# 2-opt kernels (tensor cores): launch lists of configs 2 / 5 and one full capture each
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches_c2.csv python bench.py --preset config2 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/m/ncu_launch_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m/launches_c5.csv python bench.py --preset config5 --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/m/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:twoopt_tc -s 2 -c 1 -o gpurun_out/m/prof_twoopt_c5 python bench.py --preset config5 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/m/ncu_to5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:twoopt_tc -s 2 -c 1 -o gpurun_out/m/prof_twoopt_c2 python bench.py --preset config2 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/m/ncu_to2.log 2>&1
bash scripts/gpu_velocity_sweep.sh > gpurun_out/m/velocity_sweep.log 2>&1
