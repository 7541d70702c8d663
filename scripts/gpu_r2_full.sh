# full GPU suite + smoke + config-5 / config-2 / config-3 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/full
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/full/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/full/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full/pytest_gpu.log
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/full/c5.json 2> gpurun_out/full/c5.err
timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu > gpurun_out/full/c2.json 2> gpurun_out/full/c2.err
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/full/c3.json 2> gpurun_out/full/c3.err
tail -1 gpurun_out/full/smoke.log; tail -2 gpurun_out/full/pytest_gpu.log
for f in c5 c2 c3; do python -c "
import json; d=json.load(open('gpurun_out/full/$f.json')); r2=d.get('roofline_twoopt') or {}
print('$f', round(d['value']), d['ms_per_step'], 'frac', round(d['roofline']['frac'],3), '2opt', r2.get('kernel_ms'), r2.get('frac'))"; done
