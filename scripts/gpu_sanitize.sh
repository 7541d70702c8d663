# compute-sanitizer over every kernel family at tiny sizes (scripts/sanitize_cases.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize_cases.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/summary.txt
done
cat gpurun_out/sanitize/summary.txt
