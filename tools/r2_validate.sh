# TMA GEMM validation: pipeline check (TMA vs cp.async on every routed GEMM), rank determinism,
# numerics tests, shape timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2n
for pr in "4 3 exp_neg_r 16000" "4 3 one_over_r 32000" "3 2 one_over_r 32768" "4 2 log_r 16000"; do
  echo "== check $pr"; HB_GEMM_CHECK=1 timeout 300 python tools/solo.py $pr 1 2>&1 | grep -c "gemm check"
  timeout 300 python tools/solo.py $pr 3 2>&1 | grep problem | cut -c1-110
done
for i in 1 2 3; do timeout 120 python tools/gemm_repro2.py 14440 14320 120 16000 2>&1 | grep -v Warn | head -3 | cut -c1-90; done
timeout 120 python tools/gemm_repro2.py 10600 10480 117 16000 2>&1 | grep -v Warn | head -3 | cut -c1-90
timeout 600 python tools/gemm_determinism.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_entries.py -q -x -k gemm 2>&1 | tail -2
timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing|cert"
