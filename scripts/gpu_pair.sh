# CTA-pair 2-opt: parity tests, then config 5 with the one-SM (tcp) and pair kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pair
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "twoopt" -x > gpurun_out/pair/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pair/pytest.log
tail -3 gpurun_out/pair/pytest.log
if grep -q "rc=0" gpurun_out/pair/pytest.log; then
  for k in tcp pair; do
    if [ $k = pair ]; then export QSB_TWOOPT_KERNEL=pair; else unset QSB_TWOOPT_KERNEL; fi
    timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/pair/c5_$k.json 2> gpurun_out/pair/c5_$k.err
    python -c "
import json; d=json.load(open('gpurun_out/pair/c5_$k.json')); r=d['roofline_twoopt']; print('$k', round(d['value']), d['ms_per_step'], r['kernel_ms'], round(r['frac'],3), d['best_cost'])"
  done
fi
