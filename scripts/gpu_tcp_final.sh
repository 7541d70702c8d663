# pipelined 2-opt after the round-2 tuning: GPU suite, config-5 bench line, ncu capture + launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tf
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tf/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tf/pytest.log
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/tf/bench_config5.json 2> gpurun_out/tf/c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:twoopt_tcp -s 3 -c 1 -o gpurun_out/tf/prof_tcp python bench.py --preset config5 --steps 2 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/tf/ncu.log 2>&1
ncu -i gpurun_out/tf/prof_tcp.ncu-rep --page raw --csv > gpurun_out/tf/raw.csv 2>/dev/null
ncu -i gpurun_out/tf/prof_tcp.ncu-rep --page source --csv --print-source sass > gpurun_out/tf/sass.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/tf/launches_c5.csv python bench.py --preset config5 --steps 10 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/tf/ncu_l.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/tf/bench_config5.json')); t=d.get('roofline_twoopt'); r=d['roofline']; print('c5', round(d['value']), d['ms_per_step'], r['kernel_ms'], r['frac'], t['kernel_ms'], t['frac'], d.get('e2e'))"
