# ncu captures (cuda,sass view) of the config-4 and config-5 fused steps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mwp
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 -o gpurun_out/mwp/c4 python bench.py --preset config4 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/mwp/ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 5 -c 1 -o gpurun_out/mwp/c5 python bench.py --preset config5 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 --host-steps 0 --fp64-steps 0 > gpurun_out/mwp/ncu5.log 2>&1
for c in c4 c5; do
ncu -i gpurun_out/mwp/$c.ncu-rep --page raw --csv > gpurun_out/mwp/raw_$c.csv 2>/dev/null
ncu -i gpurun_out/mwp/$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/mwp/cs_$c.csv 2>/dev/null
done
ls -la gpurun_out/mwp
