# Validation of the TMA update GEMM with the per-tile CTA barrier: every TMA GEMM of configs[3]
# (8 passes) and of the sweep (1 pass) compared with the cp.async kernel under the 4 concurrent
# sweep streams; repro without the barrier; timings; parity with the TMA kernel on
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 1500 python bench.py --steps 8 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tmaval_c3.json 2> gpurun_out/r2s3/tmaval_c3.err
echo "c3 x8 check: rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tmaval_c3.err) FRO-flags $(grep -c 'gemm check\] FRO' gpurun_out/r2s3/tmaval_c3.err)"
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_TILE_SYNC=0 timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tmaval_nosync.json 2> gpurun_out/r2s3/tmaval_nosync.err
echo "c3 x1 check, no barrier: rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tmaval_nosync.err)"
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 timeout 1800 python bench.py --workload sweep --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tmaval_sweep.json 2> gpurun_out/r2s3/tmaval_sweep.err
echo "sweep x1 check: rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tmaval_sweep.err) FRO-flags $(grep -c 'gemm check\] FRO' gpurun_out/r2s3/tmaval_sweep.err)"
HB_GEMM_TMA=1 timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing|cert" > gpurun_out/r2s3/gemm_bench_tma_sync.log; cat gpurun_out/r2s3/gemm_bench_tma_sync.log
HB_GEMM_TMA=1 HB_TMA_TILE_SYNC=0 timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing update A2|N=65536 \(K=120\)"
timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing update A2|N=65536 \(K=120\)"
HB_GEMM_TMA=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2s3/bench_c3_tma.json 2> gpurun_out/r2s3/bench_c3_tma.err
python -c "import json; d=json.loads(open('gpurun_out/r2s3/bench_c3_tma.json').read().strip().splitlines()[-1]); print('c3 TMA ms', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'], 'gemm', d['roofline']['kernel']['achieved'])"
HB_GEMM_TMA=1 timeout 1500 python bench.py --workload sweep --no-cpu-baseline > gpurun_out/r2s3/bench_sweep_tma.json 2> gpurun_out/r2s3/bench_sweep_tma.err
python -c "import json; d=json.loads(open('gpurun_out/r2s3/bench_sweep_tma.json').read().strip().splitlines()[-1]); print('sweep TMA ms', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
