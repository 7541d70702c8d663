# A/B: per-iteration kernel times for two builds on the same box
cd $GRAFT_REPO_ROOT
for lib in libqsb_prev.so libqsb.so libqsb_prev.so libqsb.so; do
  echo "== $lib"
  QSB_LIB=$PWD/paper_1504_05158_b200/$lib timeout 600 python scripts/diag_steps.py fp32 300 | python -c "
import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; v=list(k.values()); print('first', v[:3], 'mean', sum(v)/len(v), 'last', v[-3:])"
done
