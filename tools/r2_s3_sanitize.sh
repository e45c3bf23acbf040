# compute-sanitizer over every kernel path (small problems), then the TMA update GEMM under
# racecheck; then the sweep bench (configs[4]) and the solo time of its largest problem
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
python tools/sanitize_paths.py > gpurun_out/r2s3/sanitize_plain.log 2>&1; tail -3 gpurun_out/r2s3/sanitize_plain.log
HB_GEMM_TMA=1 python tools/sanitize_paths.py tma > gpurun_out/r2s3/sanitize_plain_tma.log 2>&1; tail -2 gpurun_out/r2s3/sanitize_plain_tma.log
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_paths.py > gpurun_out/r2s3/sanitize_$tool.log 2>&1
  echo "$tool rc $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|\[sanitize\]" gpurun_out/r2s3/sanitize_$tool.log | tail -12
done
for tool in memcheck racecheck; do
  HB_GEMM_TMA=1 timeout 900 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_paths.py tma > gpurun_out/r2s3/sanitize_tma_$tool.log 2>&1
  echo "tma $tool rc $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|\[sanitize\]" gpurun_out/r2s3/sanitize_tma_$tool.log | tail -4
done
timeout 300 python tools/solo.py 4 3 exp_neg_r 65536 2 > gpurun_out/r2s3/solo_4d3_65536.log 2>&1; tail -3 gpurun_out/r2s3/solo_4d3_65536.log
timeout 1500 python bench.py --workload sweep --details gpurun_out/r2s3/sweep_details.json > gpurun_out/r2s3/bench_sweep.json 2> gpurun_out/r2s3/bench_sweep.err; tail -c 3000 gpurun_out/r2s3/bench_sweep.json
