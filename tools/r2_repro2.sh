cd $GRAFT_REPO_ROOT
timeout 120 python tools/gemm_repro2.py 14440 14320 120 16000 2>&1 | grep -v Warn | tail -4
