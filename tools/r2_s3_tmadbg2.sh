cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
for rep in 1 2; do
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=512 timeout 1200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tmadbg2_$rep.out 2> gpurun_out/r2s3/tmadbg2_$rep.err
echo "dbg rep $rep rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tmadbg2_$rep.err) dbg $(grep -c 'tma dbg' gpurun_out/r2s3/tmadbg2_$rep.out)"
grep 'tma dbg' gpurun_out/r2s3/tmadbg2_$rep.out | head -30
grep 'gemm diag\] bad' gpurun_out/r2s3/tmadbg2_$rep.err | head -4 | cut -c1-160
done
for rep in 1 2 3; do
HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=128 timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tv3_128_$rep.json 2> gpurun_out/r2s3/tv3_128_$rep.err
echo "v128 rep $rep rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tv3_128_$rep.err)"
done
HB_GEMM_TMA=1 HB_TMA_VARIANT=128 timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing|cert" > gpurun_out/r2s3/gemm_bench_v128.log; cat gpurun_out/r2s3/gemm_bench_v128.log
HB_GEMM_TMA=1 timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "trailing|cert" > gpurun_out/r2s3/gemm_bench_v0.log; cat gpurun_out/r2s3/gemm_bench_v0.log
timeout 1500 python tools/solo_all.py gpurun_out/r2s3/solo_all.json > gpurun_out/r2s3/solo_all.log 2>&1; tail -2 gpurun_out/r2s3/solo_all.log
