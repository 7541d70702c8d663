# A/B of best_kernel block size (QSB_BEST_WPB=4 vs the default 8) after the
# batched last-block merge; GPU tests first.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/best
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/best/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/best/pytest.log
tail -2 gpurun_out/best/pytest.log
for rep in 1 2; do for w in 8 4; do
  QSB_BEST_WPB=$w timeout 600 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/best/c3_w$w.$rep.json 2>/dev/null
  QSB_BEST_WPB=$w timeout 300 python bench.py --preset config1 --no-cpu --steps 400 --graph > gpurun_out/best/c1_w$w.$rep.json 2>/dev/null
done; done
for f in gpurun_out/best/*.json; do echo "$f: $(python -c "
import json
d=json.load(open('$f')); r=d.get('roofline') or {}
print(round(d['value']), 'ms', round(d.get('ms_per_step',0),5), 'kern', r.get('kernel_ms'))")"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/best/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/best/launches.csv | grep -A3 best_kernel
