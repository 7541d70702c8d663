# pipelined 2-opt kernel: parity tests, then config 5 with the old (tc) and new kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tcp
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "twoopt" -x > gpurun_out/tcp/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tcp/pytest.log
tail -3 gpurun_out/tcp/pytest.log
if grep -q "rc=0" gpurun_out/tcp/pytest.log; then
  QSB_TWOOPT_KERNEL=tc timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/tcp/c5_tc.json 2> gpurun_out/tcp/c5_tc.err
  timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/tcp/c5_tcp.json 2> gpurun_out/tcp/c5_tcp.err
  for f in c5_tc c5_tcp; do python -c "
import json; d=json.load(open('gpurun_out/tcp/$f.json')); print('$f', round(d['value']), d['ms_per_step'], d.get('roofline_twoopt'))"; done
fi
