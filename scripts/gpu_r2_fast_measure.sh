# config 3 over iterations 21-420, per-iteration kernel times, early / late ncu captures, launch list, strong proxy
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fm gpurun_out/sp
timeout 600 python bench.py --steps 400 --warmup 20 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/fm/config3_400.json 2> gpurun_out/fm/config3_400.err
timeout 300 python scripts/diag_steps.py fp32 500 > gpurun_out/fm/steps.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 9 -c 1 -o gpurun_out/fm/prof_t10 python scripts/diag_steps.py fp32 11 > gpurun_out/fm/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 300 -c 1 -o gpurun_out/fm/prof_t301 python scripts/diag_steps.py fp32 302 > gpurun_out/fm/ncu2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fm/launches_c3.csv python bench.py --steps 20 --warmup 5 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/fm/ncu_c3.log 2>&1
bash scripts/gpu_strong_proxy.sh > gpurun_out/fm/strong_proxy.txt 2>&1
cat gpurun_out/fm/strong_proxy.txt; python -c "
import json; d=json.load(open('gpurun_out/fm/config3_400.json')); print('c3_400', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
