# round 2: sanitizers, per-iteration kernel times and fresh early/late ncu captures of the fused step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2prof
timeout 300 python scripts/diag_steps.py fp32 500 > gpurun_out/r2prof/steps.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 9 -c 1 -o gpurun_out/r2prof/prof_early python scripts/diag_steps.py fp32 11 > gpurun_out/r2prof/ncu_early.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 300 -c 1 -o gpurun_out/r2prof/prof_late python scripts/diag_steps.py fp32 302 > gpurun_out/r2prof/ncu_late.log 2>&1
bash scripts/gpu_sanitize.sh
