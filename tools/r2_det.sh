cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2j
timeout 600 python tools/gemm_determinism.py > gpurun_out/r2j/det.log 2>&1; tail -12 gpurun_out/r2j/det.log
timeout 300 python tools/solo.py 4 3 exp_neg_r 16000 3 > gpurun_out/r2j/solo32k.log 2>&1; cat gpurun_out/r2j/solo32k.log
HB_GEMM_TMA=0 timeout 300 python tools/solo.py 4 3 exp_neg_r 16000 2 > gpurun_out/r2j/solo32k_old.log 2>&1; cat gpurun_out/r2j/solo32k_old.log
