# ncu capture (cuda,sass source view) of the n <= 32 four-particle 2-opt kernel at config 2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tc4p
timeout 600 ncu --set full --clock-control none --import-source on -k regex:twoopt_tc4 -s 5 -c 1 -o gpurun_out/tc4p/prof python bench.py --preset config2 --steps 3 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/tc4p/ncu.log 2>&1
ncu -i gpurun_out/tc4p/prof.ncu-rep --page raw --csv > gpurun_out/tc4p/raw.csv 2>/dev/null
ncu -i gpurun_out/tc4p/prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/tc4p/cs.csv 2>/dev/null
tail -1 gpurun_out/tc4p/ncu.log
