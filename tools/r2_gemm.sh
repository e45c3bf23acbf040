# TMA GEMM bring-up: numerics tests, old vs new timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_gpu_entries.py -q -x -k "gemm" > gpurun_out/r2g/pytest_gemm.log 2>&1; tail -3 gpurun_out/r2g/pytest_gemm.log
timeout 300 python tools/gemm_bench.py 5 > gpurun_out/r2g/gemm_new.log 2>&1; cat gpurun_out/r2g/gemm_new.log
timeout 300 python tools/solo.py 4 3 exp_neg_r 65536 1 > gpurun_out/r2g/solo_4d3_exp.log 2>&1; cat gpurun_out/r2g/solo_4d3_exp.log
