# A/B of the rolled-loop (I-cache footprint) variants + the parity suite on the current build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
bash scripts/gpu_ab_steps.sh "$@" > gpurun_out/ab/summary.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/ab/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu.log
cat gpurun_out/ab/summary.txt; tail -3 gpurun_out/ab/pytest_gpu.log
