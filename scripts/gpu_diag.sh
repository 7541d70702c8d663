cd $GRAFT_REPO_ROOT
timeout 600 python scripts/diag_steps.py fp32 500 > gpurun_out/diag_fp32.json 2>&1
timeout 600 python scripts/diag_steps.py fp64 300 > gpurun_out/diag_fp64.json 2>&1
timeout 300 python scripts/diag_steps.py fp32 330 80 > gpurun_out/diag_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 320 -c 1 -o gpurun_out/prof_late python scripts/diag_steps.py fp32 330 80 > gpurun_out/ncu_late.log 2>&1
cat gpurun_out/diag_fp32.json gpurun_out/diag_fp64.json; tail -2 gpurun_out/ncu_late.log
