# configs[3]: TMA GEMM on/off, serial vs 4 streams
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_rank.py -q -x -k baseline_configs > gpurun_out/r2p/pytest.log 2>&1; tail -2 gpurun_out/r2p/pytest.log
for v in "HB_GEMM_TMA=1" "HB_GEMM_TMA=0" "HB_SUBSTREAMS=1" "HB_SUBSTREAMS=2"; do
  env $v timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2p/c3.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r2p/c3.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'], d['roofline']['frac'])"
done
