cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2v
HB_NO_PRIORITY=1 HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2v/c3.json 2>gpurun_out/r2v/c3.err
echo "no-priority:"; grep -c "gemm check" gpurun_out/r2v/c3.err
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2v/c3b.json 2>gpurun_out/r2v/c3b.err
echo "priority:"; grep -c "gemm check" gpurun_out/r2v/c3b.err
