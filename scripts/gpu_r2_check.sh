# round 2 (re-entry): new tests, the full GPU suite, both bench arms at the driver's window
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_host_step.py tests/test_gpu_reference_api.py tests/test_gpu_parity_configs.py -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench20.json 2> gpurun_out/bench20.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench20_ref.json 2> gpurun_out/bench20_ref.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_new.log; tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench20.json
