cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/vp
timeout 300 python bench.py --velocity-only --no-cpu --steps 20 --warmup 3 > gpurun_out/vp/v50.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o /tmp/vp python bench.py --velocity-only --steps 3 --warmup 2 --no-cpu > gpurun_out/vp/ncu.log 2>&1
ncu -i /tmp/vp.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/vp/src.csv 2>/dev/null
ncu -i /tmp/vp.ncu-rep --page raw --csv > gpurun_out/vp/raw.csv 2>/dev/null
ncu -i /tmp/vp.ncu-rep --page details > gpurun_out/vp/details.txt 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/vp/v50.json')); r=d['roofline']; print('v50 kern', r['kernel_ms'], 'frac', r['frac'])"
