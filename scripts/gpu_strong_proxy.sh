# Strong-scaling proxy on one GPU: config 3 with the per-rank particle count
# of N = 1, 2, 4, 8 GPUs (800 / 400 / 200 / 100 swarms of 100).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sp
for m in 800 400 200 100; do
  timeout 600 python bench.py --no-cpu --swarms $m > gpurun_out/sp/m$m.json 2>/dev/null
done
for f in gpurun_out/sp/m800.json gpurun_out/sp/m400.json gpurun_out/sp/m200.json gpurun_out/sp/m100.json; do echo "$f: $(python -c "
import json
d=json.load(open('$f')); r=d.get('roofline') or {}
print(round(d['value']), 'ms', round(d.get('ms_per_step',0),5), 'kern', r.get('kernel_ms'), 'e2e', round((d.get('e2e') or {}).get('value') or 0), d['config'].get('l2'))")"; done
