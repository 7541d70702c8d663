cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/late
timeout 300 python scripts/diag_steps.py fp32 500 > gpurun_out/late/steps.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 300 -c 1 -o gpurun_out/late/prof_late python scripts/diag_steps.py fp32 302 > gpurun_out/late/ncu_late.log 2>&1
tail -1 gpurun_out/late/ncu_late.log
