# round 2: bench lines of every preset (configs 2-5) and an ncu capture of the config-3 fused step at t = 10
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lines
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/lines/config5.json 2> gpurun_out/lines/config5.err
timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu > gpurun_out/lines/config2.json 2> gpurun_out/lines/config2.err
timeout 300 python bench.py --preset config4 --steps 30 --warmup 3 --no-cpu > gpurun_out/lines/config4.json 2> gpurun_out/lines/config4.err
timeout 300 python bench.py --preset config1 --steps 50 --warmup 5 --no-cpu > gpurun_out/lines/config1.json 2> gpurun_out/lines/config1.err
timeout 600 python bench.py --steps 400 --warmup 20 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/lines/config3_400.json 2> gpurun_out/lines/config3_400.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 9 -c 1 -o gpurun_out/lines/prof_c3_t10 python scripts/diag_steps.py fp32 11 > gpurun_out/lines/ncu.log 2>&1
for c in config1 config2 config3_400 config4 config5; do python -c "
import json; d=json.load(open('gpurun_out/lines/$c.json')); r=d.get('roofline') or {}; t=d.get('roofline_twoopt') or {}
print('$c', round(d['value']), d['ms_per_step'], r.get('kernel_ms'), r.get('frac'), t.get('kernel_ms'), t.get('frac'))"; done
