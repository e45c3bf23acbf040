cd $GRAFT_REPO_ROOT
HB_DEBUG_STOP=1 timeout 300 python tools/solo.py 4 3 exp_neg_r 65536 1 2>&1 | grep -E "predict|problem|stop\]" | tail -12
HB_DEBUG_STOP=1 timeout 300 python tools/solo.py 4 2 exp_neg_r 65536 1 2>&1 | grep -E "predict|problem" | tail -6
HB_DEBUG_STOP=1 timeout 300 python tools/solo.py 4 3 exp_neg_r 32000 1 2>&1 | grep -E "predict|problem" | tail -6
HB_PREDICT_OPEN=0 timeout 300 python tools/solo.py 4 3 exp_neg_r 65536 1 2>&1 | grep -E "problem" | tail -2
