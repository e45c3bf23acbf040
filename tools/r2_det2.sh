cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2i
for mode in 0 1 2; do
  echo "mode $mode" >> gpurun_out/r2i/det.log
  HB_GEMM_TMA_MODE=$mode timeout 300 python tools/solo.py 4 3 exp_neg_r 16000 3 2>&1 | grep problem | cut -c1-120 >> gpurun_out/r2i/det.log
done
echo "old" >> gpurun_out/r2i/det.log
HB_GEMM_TMA=0 timeout 300 python tools/solo.py 4 3 exp_neg_r 16000 2 2>&1 | grep problem | cut -c1-120 >> gpurun_out/r2i/det.log
cat gpurun_out/r2i/det.log
