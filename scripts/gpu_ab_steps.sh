# A/B of per-iteration kernel times (config 3, 500 iterations) between libqsb.so and the variant libraries given as args
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
for lib in libqsb.so "$@"; do
  QSB_LIB=$PWD/paper_1504_05158_b200/$lib timeout 300 python scripts/diag_steps.py fp32 500 > gpurun_out/ab/$lib.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/ab/$lib.json')); k=d['kernel_ms']
print('$lib', 'wall', round(d['wall_ms_per_step'],4), 'kernel', {t:k[t] for t in ['21','101','201','301','401','481']})"
done
