cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e2e
for rep in 1 2; do
timeout 600 python bench.py --no-cpu > gpurun_out/e2e/c3.$rep.json 2>gpurun_out/e2e/err.log
timeout 300 python bench.py --preset config2 --no-cpu --steps 200 > gpurun_out/e2e/c2.$rep.json 2>>gpurun_out/e2e/err.log
done
timeout 300 python bench.py --preset config5 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/e2e/c5.json 2>>gpurun_out/e2e/err.log
for f in gpurun_out/e2e/*.json; do echo "$f: $(python -c "
import json
d=json.load(open('$f')); r=d.get('roofline') or {}
print(round(d['value']), 'ms', round(d.get('ms_per_step',0),4), 'kern', r.get('kernel_ms'), 'e2e', round((d.get('e2e') or {}).get('value') or 0))")"; done
tail -3 gpurun_out/e2e/err.log
