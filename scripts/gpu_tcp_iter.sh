# pipelined 2-opt iteration: parity tests, config-5 bench, pipeline stamps (libqsb_tt.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ti
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "twoopt" -x > gpurun_out/ti/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ti/pytest.log
tail -2 gpurun_out/ti/pytest.log
timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu > gpurun_out/ti/c5.json 2> gpurun_out/ti/c5.err
python -c "
import json; d=json.load(open('gpurun_out/ti/c5.json')); t=d.get('roofline_twoopt'); print('c5', round(d['value']), d['ms_per_step'], t['kernel_ms'], t['frac'])"
[ -f paper_1504_05158_b200/libqsb_tt.so ] && timeout 120 python scripts/tcp_timing.py > gpurun_out/ti/stamps.txt 2>&1; tail -4 gpurun_out/ti/stamps.txt
QSB_TCP_TS=0 timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ti/c5_ss.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ti/c5_ss.json')); t=d.get('roofline_twoopt'); print('c5 ss', round(d['value']), d['ms_per_step'], t['kernel_ms'], t['frac'])"
