cd $GRAFT_REPO_ROOT
bash scripts/gpu_pair.sh
timeout 300 python scripts/pair_timing.py 2>&1 | tail -4
