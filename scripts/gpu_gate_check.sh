# gated timed window: GPU suite, the driver's bench command three times, configs 1 / 2 / 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gate
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gate/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gate/pytest.log
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/gate/c3_$rep.json 2> gpurun_out/gate/c3_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/gate/c3_$rep.json')); r=d['roofline']; print('c3', round(d['value']), d['ms_per_step'], r['kernel_ms'], round(r['frac'],3), round(d['e2e']['value']), d['config']['timed_window'][:40])" || tail -3 gpurun_out/gate/c3_$rep.err
done
for pr in config2 config5; do
  timeout 300 python bench.py --preset $pr --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/gate/$pr.json 2> gpurun_out/gate/$pr.err
  python -c "
import json; d=json.load(open('gpurun_out/gate/$pr.json')); r=d['roofline']; print('$pr', round(d['value']), d['ms_per_step'], r['kernel_ms'])" || tail -3 gpurun_out/gate/$pr.err
done
timeout 300 python bench.py --preset config1 --steps 200 --warmup 10 --no-cpu --graph > gpurun_out/gate/c1.json 2> gpurun_out/gate/c1.err
python -c "
import json; d=json.load(open('gpurun_out/gate/c1.json')); print('c1', round(d['value']), d['ms_per_step'])" || tail -3 gpurun_out/gate/c1.err
