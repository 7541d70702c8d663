# ncu of the fused step kernel at a late iteration for two builds
cd $GRAFT_REPO_ROOT
for lib in libqsb_prev libqsb; do
  QSB_LIB=$PWD/paper_1504_05158_b200/$lib.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 300 -c 1 -o gpurun_out/late_$lib python scripts/diag_steps.py fp32 302 > gpurun_out/ncu_late_$lib.log 2>&1
  tail -1 gpurun_out/ncu_late_$lib.log
done
