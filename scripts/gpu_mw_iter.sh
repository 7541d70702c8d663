# multi-warp step kernel iteration: GPU suite, config 4 / 5 bench lines (two reps)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mwi
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/mwi/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/mwi/pytest.log
for rep in 1 2; do
  for pr in config4 config5; do
    timeout 300 python bench.py --preset $pr --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/mwi/$pr.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/mwi/$pr.json')); r=d['roofline']; t=d.get('roofline_twoopt') or {}; print('$pr', round(d['value']), d['ms_per_step'], r['kernel_ms'], t.get('kernel_ms'))"
  done
done
