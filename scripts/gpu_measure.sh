cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.txt 2>&1
lscpu | head -20 > gpurun_out/cpu_info.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --precision fp64 --no-cpu --steps 200 > gpurun_out/bench_fp64.json 2>> gpurun_out/bench.err
for P in 20 100 400; do timeout 300 python bench.py --n 100 --swarms $P --velocity-only --no-cpu --steps 100 > gpurun_out/bench_vel100_P${P}00.json 2>> gpurun_out/bench.err; done
timeout 300 python bench.py --velocity-only --no-cpu --steps 100 > gpurun_out/bench_vel50.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 1 -o gpurun_out/prof_step python bench.py --steps 8 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_vel50 python bench.py --velocity-only --steps 3 --warmup 2 --no-cpu > gpurun_out/ncu_vel.log 2>&1
cat gpurun_out/bench.json; tail -2 gpurun_out/bench.err
