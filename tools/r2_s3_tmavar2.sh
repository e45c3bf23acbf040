cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2s3/tv2_$name.json 2> gpurun_out/r2s3/tv2_$name.err
  echo "$name rc $? C-flags $(grep -c 'gemm check\] C' gpurun_out/r2s3/tv2_$name.err) FRO-flags $(grep -c 'gemm check\] FRO' gpurun_out/r2s3/tv2_$name.err)"
  python -c "import json; d=json.loads(open('gpurun_out/r2s3/tv2_$name.json').read().strip().splitlines()[-1]); print(' ms', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
}
run control HB_GEMM_TMA=1 HB_GEMM_CHECK=2
run v32 HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=32
run v64 HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=64
run v128 HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=128
run v0serial HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_SUBSTREAMS=1
grep 'gemm diag\] bad' gpurun_out/r2s3/tv2_v0serial.err | head -3 | cut -c1-300
timeout 1500 python tools/predict_scaling.py gpurun_out/r2s3/predict_scaling.json > gpurun_out/r2s3/predict_scaling.log 2>&1; tail -16 gpurun_out/r2s3/predict_scaling.log
