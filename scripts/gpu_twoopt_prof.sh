cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tp
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/tp/c2.csv python bench.py --preset config2 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/tp/c2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__shared_mem_per_block_dynamic --clock-control none --csv --log-file gpurun_out/tp/c5.csv python bench.py --preset config5 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/tp/c5.log 2>&1
grep -h twoopt gpurun_out/tp/c2.csv | head -14
grep -h twoopt gpurun_out/tp/c5.csv | head -6
