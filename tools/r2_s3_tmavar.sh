# TMA update GEMM under the 4 concurrent sweep streams of configs[3]: count the updates whose
# result differs from the cp.async kernel's (HB_GEMM_CHECK=1) per experiment variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
for v in 0 1 2 8 4 16 3; do
  HB_GEMM_TMA=1 HB_GEMM_CHECK=1 HB_TMA_VARIANT=$v timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2s3/tmavar_$v.json 2> gpurun_out/r2s3/tmavar_$v.err
  echo "variant $v rc $? flagged $(grep -c 'gemm check' gpurun_out/r2s3/tmavar_$v.err)"
  grep 'gemm check' gpurun_out/r2s3/tmavar_$v.err | head -3 | cut -c1-200
  python -c "import json; d=json.loads(open('gpurun_out/r2s3/tmavar_$v.json').read().strip().splitlines()[-1]); print(' ms', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
done
