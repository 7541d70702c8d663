# GPU tests + quick bench lines of every config + velocity-only n=50/100/256 (no ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ca
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ca/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ca/pytest.log
tail -2 gpurun_out/ca/pytest.log; grep -E "^FAILED|Error" gpurun_out/ca/pytest.log | head -10
timeout 300 python bench.py --no-cpu --e2e-steps 50 > gpurun_out/ca/c3.json 2>/dev/null
timeout 300 python bench.py --preset config2 --no-cpu --steps 200 > gpurun_out/ca/c2.json 2>/dev/null
timeout 300 python bench.py --preset config4 --no-cpu --steps 100 > gpurun_out/ca/c4.json 2>/dev/null
timeout 300 python bench.py --preset config5 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/ca/c5.json 2>/dev/null
timeout 300 python bench.py --velocity-only --no-cpu --steps 50 --warmup 5 > gpurun_out/ca/v50.json 2>/dev/null
timeout 300 python bench.py --preset config4 --velocity-only --no-cpu --steps 50 --warmup 5 > gpurun_out/ca/v100.json 2>/dev/null
timeout 300 python bench.py --preset config5 --velocity-only --no-cpu --steps 20 --warmup 3 > gpurun_out/ca/v256.json 2>/dev/null
for f in gpurun_out/ca/*.json; do echo "$f $(python -c "
import json; d=json.load(open('$f')); r=d['roofline']; e=d.get('e2e') or {}; print(round(d['value']), 'ms', round(d['ms_per_step'],4), 'kern', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), 'e2e', e.get('value'))")"; done
