cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gt/pytest.log
tail -2 gpurun_out/gt/pytest.log
timeout 300 python bench.py --preset config5 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/gt/c5.json 2>/dev/null
timeout 300 python bench.py --preset config5 --velocity-only --no-cpu --steps 20 --warmup 3 > gpurun_out/gt/v256.json 2>/dev/null
timeout 300 python bench.py --preset config4 --no-cpu --steps 100 > gpurun_out/gt/c4.json 2>/dev/null
timeout 300 python bench.py --preset config4 --velocity-only --no-cpu --steps 50 > gpurun_out/gt/v100.json 2>/dev/null
for f in gpurun_out/gt/*.json; do echo "$f $(python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print(round(d['value']), 'ms', round(d['ms_per_step'],4), 'kern', round(r['kernel_ms'],4), 'frac', round(r['frac'],3))")"; done
