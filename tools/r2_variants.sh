cd $GRAFT_REPO_ROOT
for v in "HB_TMA_PLAINC=1" "HB_TMA_WSC=1" "HB_TMA_PLAINC=1 HB_TMA_WSC=1"; do
  echo "== $v"
  env $v timeout 120 python tools/gemm_repro2.py 14440 14320 120 16000 2>&1 | grep -v Warn | head -3 | cut -c1-90
  env $v timeout 300 python tools/gemm_bench.py 5 2>&1 | grep "trailing update A2" | head -1
done
