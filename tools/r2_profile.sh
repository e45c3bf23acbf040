# round-2 evidence: GPU tests, ncu capture of the TMA update GEMM, launch list of one solo problem
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2q
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2q/pytest.log 2>&1; tail -3 gpurun_out/r2q/pytest.log
python tools/gemm_one.py 0 32768 32768 120 1.0 -1.0 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 1 -c 1 -o gpurun_out/r2q/tma_update python tools/gemm_one.py 0 32768 32768 120 1.0 -1.0 > gpurun_out/r2q/ncu_full.log 2>&1; tail -1 gpurun_out/r2q/ncu_full.log
python tools/solo.py 4 3 exp_neg_r 16000 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q/launches_solo_4d3_16000.csv python tools/solo.py 4 3 exp_neg_r 16000 1 > gpurun_out/r2q/ncu_list.log 2>&1; tail -1 gpurun_out/r2q/ncu_list.log
