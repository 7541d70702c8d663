# A/B of per-iteration kernel times (config 3, 500 iterations) between env settings given as args ("NAME=VAL" or "-")
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
for kv in "$@"; do
  if [ "$kv" = "-" ]; then env_set=""; else env_set="$kv"; fi
  env $env_set timeout 300 python scripts/diag_steps.py fp32 500 > gpurun_out/ab/env_$kv.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/ab/env_$kv.json')); k=d['kernel_ms']
print('$kv', 'wall', round(d['wall_ms_per_step'],4), 'kernel', {t:k[t] for t in ['21','101','201','301','401','481']})"
done
