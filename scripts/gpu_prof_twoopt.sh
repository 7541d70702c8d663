cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t
timeout 600 ncu --set full --clock-control none --import-source on -k regex:twoopt -s 3 -c 1 -o gpurun_out/t/twoopt_cfg5 python bench.py --preset config5 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/t/ncu5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:twoopt -s 5 -c 1 -o gpurun_out/t/twoopt_cfg2 python bench.py --preset config2 --no-cpu --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/t/ncu2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t/launches2.csv python bench.py --preset config2 --no-cpu --steps 20 --warmup 3 --e2e-steps 0 > /dev/null 2>&1
tail -1 gpurun_out/t/ncu5.log gpurun_out/t/ncu2.log
