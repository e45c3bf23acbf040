# final-state check on one box: GPU tests, smoke, default bench (driver flags), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3f
timeout 2400 python -m pytest tests -q -m gpu -x --durations=6 > gpurun_out/r2s3f/pytest.log 2>&1; tail -12 gpurun_out/r2s3f/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3f/smoke.log 2>&1; cat gpurun_out/r2s3f/smoke.log
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2s3f/bench_c3.json 2> gpurun_out/r2s3f/bench_c3.err; tail -c 1500 gpurun_out/r2s3f/bench_c3.json
timeout 600 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2s3f/bench_c3_ref.json 2> gpurun_out/r2s3f/bench_c3_ref.err; tail -c 600 gpurun_out/r2s3f/bench_c3_ref.json
