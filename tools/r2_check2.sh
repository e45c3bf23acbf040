cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2k
HB_GEMM_CHECK=1 timeout 300 python tools/solo.py 4 3 exp_neg_r 16000 2 > gpurun_out/r2k/check.log 2>&1
grep -c "gemm check" gpurun_out/r2k/check.log; grep "gemm check" gpurun_out/r2k/check.log | head -20; grep problem gpurun_out/r2k/check.log | cut -c1-150
