cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tmadiag.json 2> gpurun_out/r2s3/tmadiag.err
echo "rc $? flagged $(grep -c 'gemm check' gpurun_out/r2s3/tmadiag.err)"
grep 'gemm diag' gpurun_out/r2s3/tmadiag.err | head -40 | cut -c1-420
timeout 1500 python tools/predict_scaling.py gpurun_out/r2s3/predict_scaling.json > gpurun_out/r2s3/predict_scaling.log 2>&1; tail -12 gpurun_out/r2s3/predict_scaling.log
