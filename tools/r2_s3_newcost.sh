cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2s3/bench_c3_newcost.json 2> gpurun_out/r2s3/bench_c3_newcost.err
python -c "import json; d=json.loads(open('gpurun_out/r2s3/bench_c3_newcost.json').read().strip().splitlines()[-1]); print('c3 ms', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
timeout 1500 python bench.py --workload sweep --no-cpu-baseline > gpurun_out/r2s3/bench_sweep_newcost.json 2> gpurun_out/r2s3/bench_sweep_newcost.err
python -c "import json; d=json.loads(open('gpurun_out/r2s3/bench_sweep_newcost.json').read().strip().splitlines()[-1]); print('sweep ms', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
timeout 1500 python tools/predict_scaling.py gpurun_out/r2s3/predict_scaling_newcost.json > gpurun_out/r2s3/predict_scaling_newcost.log 2>&1; grep "^N=" gpurun_out/r2s3/predict_scaling_newcost.log | grep -v share
