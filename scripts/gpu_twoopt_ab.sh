# config 2 / config 5 bench lines with the tensor-core 2-opt (default) and the dp4a kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t
for k in tc dp4a; do
  QSB_TWOOPT_KERNEL=$k timeout 300 python bench.py --preset config2 --no-cpu --steps 200 > gpurun_out/t/c2_$k.json 2> gpurun_out/t/err.log
  QSB_TWOOPT_KERNEL=$k timeout 300 python bench.py --preset config5 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/t/c5_$k.json 2>> gpurun_out/t/err.log
done
for f in gpurun_out/t/*.json; do echo "$f $(python -c "
import json; d=json.load(open('$f')); print(round(d['value']), 'ms', round(d['ms_per_step'],4), 'kern', round(d['roofline']['kernel_ms'],4), 'e2e', round(d['e2e']['value']))")"; done
tail -3 gpurun_out/t/err.log
