# GPU suite + bench lines of configs 2-5 (config 3 at the driver's window)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/all
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/all/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/all/pytest_gpu.log; tail -2 gpurun_out/all/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/all/config3.json 2> gpurun_out/all/config3.err
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/all/config5.json 2> gpurun_out/all/config5.err
timeout 300 python bench.py --preset config4 --steps 30 --warmup 3 --no-cpu > gpurun_out/all/config4.json 2> gpurun_out/all/config4.err
timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu > gpurun_out/all/config2.json 2> gpurun_out/all/config2.err
for c in config3 config5 config4 config2; do python -c "
import json; d=json.load(open('gpurun_out/all/$c.json')); r=d.get('roofline') or {}; t=d.get('roofline_twoopt') or {}
print('$c', round(d['value']), round(d['ms_per_step'],4), round(r.get('kernel_ms') or 0,4), round(r.get('frac') or 0,3), t.get('kernel_ms'), d.get('best_cost'))"; done
