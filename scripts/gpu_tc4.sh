cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tc4
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "twoopt or graph" -x > gpurun_out/tc4/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tc4/pytest.log; tail -2 gpurun_out/tc4/pytest.log
timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/tc4/c2.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/tc4/c2.json')); print('c2', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline_twoopt']['kernel_ms'])"
