cd $GRAFT_REPO_ROOT
timeout 300 python scripts/diag_steps.py fp32 355 > gpurun_out/diag_late.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 350 -c 1 -o gpurun_out/prof_late python scripts/diag_steps.py fp32 355 > gpurun_out/ncu_late.log 2>&1
tail -2 gpurun_out/ncu_late.log
