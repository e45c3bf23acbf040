# round-2 check: GPU tests, smoke, solo of the costliest problem, default bench (configs[3])
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2o
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2o/pytest.log 2>&1; tail -3 gpurun_out/r2o/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o/smoke.log 2>&1; tail -1 gpurun_out/r2o/smoke.log
timeout 300 python tools/solo.py 4 3 exp_neg_r 65536 1 > gpurun_out/r2o/solo65k.log 2>&1; cat gpurun_out/r2o/solo65k.log
HB_TIMELINE=1 timeout 900 python bench.py --steps 2 --warmup 1 --details gpurun_out/r2o/c3_details.json > gpurun_out/r2o/bench_c3.json 2> gpurun_out/r2o/bench_c3.err; tail -c 2500 gpurun_out/r2o/bench_c3.json
