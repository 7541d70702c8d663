cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED" gpurun_out/pytest_gpu.log | head -5; tail -2 gpurun_out/pytest_gpu.log
bash scripts/ab.sh
