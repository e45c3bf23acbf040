cd $GRAFT_REPO_ROOT
for m in tma tma none; do HB_GEMM_TMA=1 timeout 300 python tools/tma_conc.py $m 60 2>&1 | grep -E "mode|Error" | head -3; done
