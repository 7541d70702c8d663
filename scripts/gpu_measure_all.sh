cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/m
timeout 900 python bench.py > gpurun_out/m/bench_config3.json 2> gpurun_out/m/err.log; echo "config3 rc=$?" >> gpurun_out/m/err.log
timeout 600 python bench.py --impl reference > gpurun_out/m/bench_reference.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config1 --no-cpu --steps 200 > gpurun_out/m/bench_config1.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config2 --no-cpu --steps 100 > gpurun_out/m/bench_config2.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --no-cpu --steps 100 > gpurun_out/m/bench_config4.json 2>> gpurun_out/m/err.log
timeout 600 python bench.py --preset config5 --no-cpu --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/m/bench_config5.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --precision fp64 --no-cpu --steps 100 > gpurun_out/m/bench_config3_fp64.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n50.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --swarms 400 --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n100_40k.json 2>> gpurun_out/m/err.log
timeout 300 python bench.py --preset config4 --velocity-only --no-cpu --steps 100 > gpurun_out/m/bench_velocity_n100_10k.json 2>> gpurun_out/m/err.log
for f in gpurun_out/m/*.json; do echo "$f: $(head -c 400 $f)"; done
tail -5 gpurun_out/m/err.log
