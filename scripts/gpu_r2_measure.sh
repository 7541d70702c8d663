# round 2: new host-step test, ncu launch list of the driver's bench command, strong-scaling proxy
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2m gpurun_out/sp
timeout 600 python -m pytest tests/test_gpu_host_step.py -q -p no:cacheprovider > gpurun_out/r2m/pytest_host.log 2>&1; echo "rc=$?" >> gpurun_out/r2m/pytest_host.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m/launches_c3.csv python bench.py --steps 20 --warmup 5 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/r2m/ncu_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m/launches_c5.csv python bench.py --preset config5 --steps 10 --warmup 3 --no-cpu --host-steps 0 --fp64-steps 0 > gpurun_out/r2m/ncu_c5.log 2>&1
bash scripts/gpu_strong_proxy.sh > gpurun_out/r2m/strong_proxy.txt 2>&1
tail -2 gpurun_out/r2m/pytest_host.log; cat gpurun_out/r2m/strong_proxy.txt
