cd $GRAFT_REPO_ROOT
bash scripts/gpu_tcp.sh
timeout 300 python scripts/tcp_timing.py 2>&1 | tail -6
