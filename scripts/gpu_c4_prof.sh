# ncu capture (cuda,sass view) of the config-4 fused step (n = 100, 4-warp groups)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c4p
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:step_kernel -s 5 -c 1 -o gpurun_out/c4p/prof python bench.py --preset config4 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/c4p/ncu.log 2>&1
ncu -i gpurun_out/c4p/prof.ncu-rep --page raw --csv > gpurun_out/c4p/raw.csv 2>/dev/null
ncu -i gpurun_out/c4p/prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c4p/cs.csv 2>/dev/null
tail -1 gpurun_out/c4p/ncu.log
