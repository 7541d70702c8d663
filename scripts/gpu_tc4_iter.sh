# n <= 32 2-opt kernel iteration: parity tests, config-2 bench (two reps)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t4
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "twoopt" -x > gpurun_out/t4/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t4/pytest.log
tail -2 gpurun_out/t4/pytest.log
for rep in 1 2; do
timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/t4/c2_$rep.json 2> gpurun_out/t4/c2.err
python -c "
import json; d=json.load(open('gpurun_out/t4/c2_$rep.json')); t=d.get('roofline_twoopt'); r=d['roofline']; print('c2', round(d['value']), d['ms_per_step'], r['kernel_ms'], t['kernel_ms'], t['frac'])"
done
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t4/c5.json 2> gpurun_out/t4/c5.err
python -c "
import json; d=json.load(open('gpurun_out/t4/c5.json')); t=d.get('roofline_twoopt'); r=d['roofline']; print('c5', round(d['value']), d['ms_per_step'], r['kernel_ms'], t['kernel_ms'], t['frac'])"
