cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=512 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tmadbg.out 2> gpurun_out/r2s3/tmadbg.err
echo "rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tmadbg.err) dbg $(grep -c 'tma dbg' gpurun_out/r2s3/tmadbg.out)"
grep 'tma dbg' gpurun_out/r2s3/tmadbg.out | head -50
grep 'gemm diag\] bad' gpurun_out/r2s3/tmadbg.err | head -3 | cut -c1-200
