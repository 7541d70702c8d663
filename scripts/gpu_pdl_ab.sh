# A/B of programmatic dependent launch (coef -> step -> best chain): GPU
# tests with PDL on, then config 3 / config 2 / config 1 bench lines with and without it.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pdl/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pdl/pytest.log
tail -2 gpurun_out/pdl/pytest.log
for rep in 1 2; do
for v in 0 1; do
  QSB_NO_PDL=$v timeout 600 python bench.py --no-cpu > gpurun_out/pdl/c3_nopdl$v.$rep.json 2>/dev/null
  QSB_NO_PDL=$v timeout 300 python bench.py --preset config2 --no-cpu --steps 200 > gpurun_out/pdl/c2_nopdl$v.$rep.json 2>/dev/null
  QSB_NO_PDL=$v timeout 300 python bench.py --preset config1 --no-cpu --steps 400 --graph > gpurun_out/pdl/c1_nopdl$v.$rep.json 2>/dev/null
done; done
for f in gpurun_out/pdl/*.json; do echo "$f: $(python -c "
import json
d=json.load(open('$f')); r=d.get('roofline') or {}
print(round(d['value']), 'ms', round(d.get('ms_per_step',0),4), 'kern', r.get('kernel_ms'), 'e2e', round((d.get('e2e') or {}).get('value') or 0))")"; done
