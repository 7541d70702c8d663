# A/B of the driver-window bench line (and iterations 21-420) between libqsb.so and libqsb_base.so, alternating
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abl
for rep in 1 2 3; do
  for lib in libqsb.so libqsb_base.so; do
    QSB_LIB=$PWD/paper_1504_05158_b200/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/abl/w.json 2>/dev/null
    QSB_LIB=$PWD/paper_1504_05158_b200/$lib timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/abl/l.json 2>/dev/null
    python -c "
import json; w=json.load(open('gpurun_out/abl/w.json')); l=json.load(open('gpurun_out/abl/l.json')); print('$lib', round(w['value']/1e6,2), round(w['roofline']['kernel_ms'],4), round(l['value']/1e6,2))"
  done
done
