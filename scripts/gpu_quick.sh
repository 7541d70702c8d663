# quick GPU check: parity tests + per-iteration kernel times over 500 iterations (config 3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/q
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/q/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest.log
tail -2 gpurun_out/q/pytest.log
timeout 300 python scripts/diag_steps.py fp32 500 > gpurun_out/q/steps.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/q/steps.json')); k=d['kernel_ms']
print('wall', round(d['wall_ms_per_step'],4), 'kernel', {t:k[t] for t in ['21','101','201','301','401','481']})"
