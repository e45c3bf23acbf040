# after the K-tail / M-tail DMMA skips: GEMM numerics tests, GEMM timings, full GPU suite, smoke,
# default bench (configs[3]), reference arm, sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3h
timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "x" > gpurun_out/r2s3h/gemm_bench.log; cat gpurun_out/r2s3h/gemm_bench.log
timeout 2400 python -m pytest tests -q -m gpu --durations=6 > gpurun_out/r2s3h/pytest.log 2>&1; tail -12 gpurun_out/r2s3h/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3h/smoke.log 2>&1; cat gpurun_out/r2s3h/smoke.log
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2s3h/bench_c3.json 2> gpurun_out/r2s3h/bench_c3.err
python -c "import json; d=json.loads(open('gpurun_out/r2s3h/bench_c3.json').read().strip().splitlines()[-1]); print('c3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel']['achieved'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'], d['clocks'])"
timeout 600 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2s3h/bench_c3_ref.json 2> gpurun_out/r2s3h/bench_c3_ref.err; tail -c 300 gpurun_out/r2s3h/bench_c3_ref.json
timeout 1500 python bench.py --workload sweep --no-cpu-baseline > gpurun_out/r2s3h/bench_sweep.json 2> gpurun_out/r2s3h/bench_sweep.err
python -c "import json; d=json.loads(open('gpurun_out/r2s3h/bench_sweep.json').read().strip().splitlines()[-1]); print('sweep', d['value'], d['ms_per_step'], d['roofline']['frac'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
