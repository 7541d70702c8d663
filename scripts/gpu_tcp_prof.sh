# ncu capture of the pipelined 2-opt kernel (config 5) with its SASS page
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tcpp
timeout 900 ncu --set full --clock-control none --import-source on -k regex:twoopt_tcp -s 3 -c 1 -o gpurun_out/tcpp/prof python bench.py --preset config5 --steps 2 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/tcpp/ncu.log 2>&1
ncu -i gpurun_out/tcpp/prof.ncu-rep --page raw --csv > gpurun_out/tcpp/raw.csv 2>/dev/null
ncu -i gpurun_out/tcpp/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/tcpp/sass.csv 2>/dev/null
tail -2 gpurun_out/tcpp/ncu.log
