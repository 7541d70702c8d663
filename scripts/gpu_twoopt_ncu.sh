cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tn
timeout 600 ncu --set full --clock-control none --import-source on -k regex:twoopt_tc -s 2 -c 1 -o gpurun_out/tn/c5 python bench.py --preset config5 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/tn/c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:twoopt_tc -s 2 -c 1 -o gpurun_out/tn/c2 python bench.py --preset config2 --no-cpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/tn/c2.log 2>&1
tail -2 gpurun_out/tn/c5.log gpurun_out/tn/c2.log
