cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
for args in "20000 19880 120 0 0 0" "20000 19880 120 1 0 0" "20000 19880 120 0 1 0" "20000 19880 120 0 0 1" "20000 19880 120 1 1 1" "4000 3000 120 1 0 1" "4000 3000 100 0 0 0"; do
  timeout 120 python tools/gemm_repro.py $args >> gpurun_out/r2d/repro.log 2>&1 || echo "FAIL $args" >> gpurun_out/r2d/repro.log
done
cat gpurun_out/r2d/repro.log | grep -v Warning | tail -30
timeout 300 compute-sanitizer --tool memcheck python tools/gemm_repro.py 4000 3000 120 1 0 1 > gpurun_out/r2d/sanitize.log 2>&1; head -60 gpurun_out/r2d/sanitize.log
