# r02 evidence for the product path (cp.async DMMA GEMM, HB_GEMM_TMA unset): ncu --set full of the
# rank-120 trailing update, and the launch list of one solo problem (after the plain runs exit 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
python tools/gemm_one.py 0 32768 32768 120 1.0 -1.0 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s 1 -c 1 -o gpurun_out/r2s3/cpasync_update python tools/gemm_one.py 0 32768 32768 120 1.0 -1.0 > gpurun_out/r2s3/ncu_full.log 2>&1; tail -1 gpurun_out/r2s3/ncu_full.log
python tools/solo.py 4 3 exp_neg_r 16000 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3/launches_solo_4d3_16000_default.csv python tools/solo.py 4 3 exp_neg_r 16000 1 > gpurun_out/r2s3/ncu_list.log 2>&1; tail -1 gpurun_out/r2s3/ncu_list.log
HB_TIMELINE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2s3/c3_timeline.json 2> gpurun_out/r2s3/c3_timeline.err; grep -c timeline gpurun_out/r2s3/c3_timeline.err
