# session-3 first call: GPU tests, smoke, default bench (configs[3]), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/pytest.log 2>&1; tail -3 gpurun_out/r2s3/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3/smoke.log 2>&1; cat gpurun_out/r2s3/smoke.log
timeout 900 python bench.py --details gpurun_out/r2s3/c3_details.json > gpurun_out/r2s3/bench_c3.json 2> gpurun_out/r2s3/bench_c3.err; tail -1 gpurun_out/r2s3/bench_c3.json
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/r2s3/bench_c3_ref.json 2> gpurun_out/r2s3/bench_c3_ref.err; tail -1 gpurun_out/r2s3/bench_c3_ref.json
