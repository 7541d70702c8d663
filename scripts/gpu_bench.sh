cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --velocity-only --no-cpu --steps 200 > gpurun_out/bench_vel50.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --n 100 --swarms 100 --velocity-only --no-cpu --steps 200 > gpurun_out/bench_vel100.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --precision fp64 --no-cpu --steps 100 > gpurun_out/bench_fp64.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 -o gpurun_out/prof_step python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
echo done
cat gpurun_out/bench.json gpurun_out/bench_vel50.json gpurun_out/bench_vel100.json gpurun_out/bench_fp64.json; tail -3 gpurun_out/bench.err; tail -3 gpurun_out/ncu_full.log
