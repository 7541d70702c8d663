cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/diag_steps.py fp32 300 > gpurun_out/diag_fp32.json 2>&1
timeout 600 python scripts/diag_steps.py fp64 100 > gpurun_out/diag_fp64.json 2>&1
timeout 300 python scripts/diag_steps.py fp32 12 > gpurun_out/diag_short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 8 -c 1 -o gpurun_out/prof_early python scripts/diag_steps.py fp32 12 > gpurun_out/ncu_early.log 2>&1
tail -4 gpurun_out/pytest_gpu.log; cat gpurun_out/diag_fp32.json gpurun_out/diag_fp64.json
timeout 600 python bench.py --no-cpu --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 1500
