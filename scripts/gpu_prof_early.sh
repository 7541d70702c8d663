cd $GRAFT_REPO_ROOT
timeout 300 python scripts/diag_steps.py fp32 12 > gpurun_out/diag_short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 8 -c 1 -o gpurun_out/prof_early python scripts/diag_steps.py fp32 12 > gpurun_out/ncu_early.log 2>&1
tail -1 gpurun_out/ncu_early.log
