# A/B: draw pre-pass folded into the previous best update (default) vs a
# separate coef_kernel per step (QSB_NO_COEF_FOLD=1); GPU suite first
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fold
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fold/pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/fold/pytest.log
for rep in 1 2; do
  for kv in "QSB_NO_COEF_FOLD=0" "QSB_NO_COEF_FOLD=1"; do
    env $kv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --host-steps 0 --fp64-steps 0 --e2e-steps 0 > gpurun_out/fold/c3_${kv}_$rep.json 2>/dev/null
    env $kv timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu --host-steps 0 --fp64-steps 0 --e2e-steps 0 > gpurun_out/fold/c3l_${kv}_$rep.json 2>/dev/null
    env $kv timeout 300 python bench.py --swarms 100 --steps 400 --warmup 20 --no-cpu --host-steps 0 --fp64-steps 0 --e2e-steps 0 > gpurun_out/fold/m100_${kv}_$rep.json 2>/dev/null
    env $kv timeout 300 python bench.py --preset config4 --steps 30 --warmup 3 --no-cpu > gpurun_out/fold/c4_${kv}_$rep.json 2>/dev/null
  done
done
for f in gpurun_out/fold/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']), d['ms_per_step'], d.get('gpu_launches'))" 2>/dev/null || echo "$f bad"; done
