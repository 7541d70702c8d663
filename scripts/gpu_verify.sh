cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/v/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/v/bench.json 2> gpurun_out/v/bench.err; echo "bench rc=$?" >> gpurun_out/v/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/v/bench_ref.json 2> gpurun_out/v/bench_ref.err
tail -2 gpurun_out/v/smoke.log; tail -3 gpurun_out/v/pytest_gpu.log; cat gpurun_out/v/bench.json | head -c 1500
