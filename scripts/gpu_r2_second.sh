# round 2: host-buffer step, reference-API restatement, full suite, benches
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_host_step.py tests/test_gpu_reference_api.py tests/test_gpu_parity_configs.py -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/pytest_new2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new2.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench20.json 2> gpurun_out/bench20.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench20_ref.json 2> gpurun_out/bench20_ref.err
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_new2.log; tail -2 gpurun_out/pytest_gpu.log
