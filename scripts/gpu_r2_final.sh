# round-2 final measurement: smoke, GPU suite, driver-window bench line (with CPU
# baseline and e2e), reference arm, every preset, config 3 over 400 iterations,
# launch lists, ncu capture of the config-3 fused step at t = 10
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fin/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin/bench_config3_driver_window.json 2> gpurun_out/fin/c3.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin/bench_reference_driver_window.json 2> gpurun_out/fin/ref.err
timeout 600 python bench.py --steps 400 --warmup 20 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/fin/bench_config3_400.json 2> gpurun_out/fin/c3_400.err
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/fin/bench_config5.json 2> gpurun_out/fin/c5.err
timeout 300 python bench.py --preset config4 --steps 30 --warmup 3 --no-cpu > gpurun_out/fin/bench_config4.json 2> gpurun_out/fin/c4.err
timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu > gpurun_out/fin/bench_config2.json 2> gpurun_out/fin/c2.err
timeout 300 python bench.py --preset config1 --steps 200 --warmup 10 --no-cpu --graph > gpurun_out/fin/bench_config1_graph.json 2> gpurun_out/fin/c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches_c3.csv python bench.py --steps 20 --warmup 5 --no-cpu --host-steps 0 --fp64-steps 0 --e2e-steps 0 > gpurun_out/fin/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 9 -c 1 -o gpurun_out/fin/prof_c3_t10 python scripts/diag_steps.py fp32 11 > gpurun_out/fin/ncu_prof.log 2>&1
ncu -i gpurun_out/fin/prof_c3_t10.ncu-rep --page raw --csv > gpurun_out/fin/raw_c3_t10.csv 2>/dev/null
bash scripts/gpu_strong_proxy.sh > gpurun_out/fin/strong_proxy.txt 2>&1; cp gpurun_out/sp/*.json gpurun_out/fin/ 2>/dev/null
for f in bench_config3_driver_window bench_reference_driver_window bench_config3_400 bench_config5 bench_config4 bench_config2 bench_config1_graph; do python -c "
import json; d=json.load(open('gpurun_out/fin/$f.json')); r=d.get('roofline') or {}; t=d.get('roofline_twoopt') or {}; e=d.get('e2e') or {}
print('$f', round(d.get('value') or 0), d.get('ms_per_step'), r.get('kernel_ms'), r.get('frac'), t.get('kernel_ms'), t.get('frac'), 'e2e', e.get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d.get('clocks',{}).get('reasons'))" 2>&1 | tail -1; done
cat gpurun_out/fin/strong_proxy.txt
