cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab2
bash scripts/gpu_ab_steps.sh libqsb_base.so libqsb_v3.so > gpurun_out/ab2/summary.txt 2>&1
timeout 600 python scripts/host_e2e_sweep.py 8 16 32 64 > gpurun_out/ab2/host_sweep.json 2>&1
cat gpurun_out/ab2/summary.txt gpurun_out/ab2/host_sweep.json
