cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/diag_steps.py fp32 400 > gpurun_out/diag_fp32.json 2>&1
grep -E "FAILED" gpurun_out/pytest_gpu.log | head -20; tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/diag_fp32.json
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/diag_steps.py fp32 12 > gpurun_out/diag_short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 8 -c 1 -o gpurun_out/prof_early python scripts/diag_steps.py fp32 12 > gpurun_out/ncu_early.log 2>&1
tail -1 gpurun_out/ncu_early.log
