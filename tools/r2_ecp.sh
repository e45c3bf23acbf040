cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2w
timeout 600 python -m pytest tests/test_gpu_entries.py -q -x -k gemm 2>&1 | tail -1
HB_GEMM_ECP=0 timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing|cert|band"
timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing|cert|band"
timeout 120 python tools/gemm_determinism.py 2>&1 | tail -2
HB_GEMM_CHECK=1 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2w/c3chk.json 2>gpurun_out/r2w/c3chk.err
echo "ecp check (concurrent c3):"; grep -c "gemm check" gpurun_out/r2w/c3chk.err; grep "gemm check" gpurun_out/r2w/c3chk.err | head -3
timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2w/c3.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r2w/c3.json').read().strip().splitlines()[-1]); p=d['parity']; print('c3', d['ms_per_step'], d['value'], d['roofline']['frac'], p['equal'], p['checked_vs_oracle'], d['roofline']['kernel']['achieved'])"
