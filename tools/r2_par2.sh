cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2u
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2u/pytest.log 2>&1; tail -2 gpurun_out/r2u/pytest.log
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2u/c3.json 2>gpurun_out/r2u/c3.err
grep -c "gemm check" gpurun_out/r2u/c3.err; grep "gemm check" gpurun_out/r2u/c3.err | head -3
HB_SUBSTREAMS=1 HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2u/c3s.json 2>gpurun_out/r2u/c3s.err
grep -c "gemm check" gpurun_out/r2u/c3s.err; grep "gemm check" gpurun_out/r2u/c3s.err | head -3
