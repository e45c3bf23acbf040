cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2f
python tools/gemm_one.py 0 32768 32768 120 1.0 -1.0 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 1 -c 1 -o gpurun_out/r2f/tma_update python tools/gemm_one.py 0 32768 32768 120 1.0 -1.0 > gpurun_out/r2f/ncu.log 2>&1
tail -3 gpurun_out/r2f/ncu.log
