# round 2: new parity tests first, then the full GPU suite and a short bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 600 -p no:cacheprovider -x -rA > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench20.json 2> gpurun_out/bench20.err
timeout 600 python bench.py --steps 400 --warmup 20 --no-cpu > gpurun_out/bench400.json 2> gpurun_out/bench400.err
tail -3 gpurun_out/pytest_new.log; tail -3 gpurun_out/pytest_gpu.log
