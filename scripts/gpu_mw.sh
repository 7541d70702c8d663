# multi-warp step kernels: parity tests, then configs 4 and 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mw
timeout 900 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/mw/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mw/pytest.log; tail -2 gpurun_out/mw/pytest.log
for c in config4 config5; do timeout 300 python bench.py --preset $c --steps 30 --warmup 3 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/mw/$c.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/mw/$c.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d.get('best_cost'))"; done
