# step-kernel iteration: GPU suite, config 3 / 4 / 5 bench lines (two reps)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ia
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ia/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ia/pytest.log
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/ia/config3.json 2>/dev/null
  timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/ia/config3l.json 2>/dev/null
  for pr in config4 config5; do
    timeout 300 python bench.py --preset $pr --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ia/$pr.json 2>/dev/null
  done
  for pr in config3 config3l config4 config5; do python -c "
import json; d=json.load(open('gpurun_out/ia/$pr.json')); r=d['roofline']; t=d.get('roofline_twoopt') or {}; print('$pr', round(d['value']), d['ms_per_step'], r['kernel_ms'], t.get('kernel_ms'))"; done
done
