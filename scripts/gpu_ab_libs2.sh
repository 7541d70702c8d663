# A/B (alternating, three reps) of libqsb.so against libqsb_base.so: config 3 window / 400 iterations, configs 2 / 4 / 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abl2
for rep in 1 2 3; do
  for lib in libqsb.so libqsb_base.so; do
    L=$PWD/paper_1504_05158_b200/$lib
    QSB_LIB=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/abl2/w.json 2>/dev/null
    QSB_LIB=$L timeout 300 python bench.py --steps 400 --warmup 20 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/abl2/l.json 2>/dev/null
    QSB_LIB=$L timeout 300 python bench.py --preset config2 --steps 100 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/abl2/c2.json 2>/dev/null
    QSB_LIB=$L timeout 300 python bench.py --preset config5 --steps 30 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/abl2/c5.json 2>/dev/null
    python -c "
import json; f=lambda x: round(json.load(open('gpurun_out/abl2/'+x+'.json'))['value']/1e6,2)
print('$lib', f('w'), f('l'), f('c2'), f('c5'))"
  done
done
