cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED" gpurun_out/pytest_gpu.log | head; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --preset config4 --no-cpu --steps 100 2>&1 | head -c 600; echo
timeout 600 python bench.py --preset config5 --no-cpu --steps 5 --warmup 3 --e2e-steps 3 --two-opt 0 2>&1 | head -c 400; echo
