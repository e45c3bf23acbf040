# c3 parity under concurrency: TMA GEMM on / off, 3 timed steps each, mismatches listed
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2t
for v in "HB_GEMM_TMA=1" "HB_GEMM_TMA=0" "HB_GEMM_TMA=1 HB_GEMM_CHECK=1"; do
  env $v timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2t/c3.json 2>gpurun_out/r2t/c3.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2t/c3.json').read().strip().splitlines()[-1]); p=d['parity']
print('$v', d['ms_per_step'], p['equal'], p['checked_vs_oracle'], p['uncertified_brackets'], p['rounding_sensitive']['count'])
for m in p['mismatches']: print('   ', m)
"
  grep -c "gemm check" gpurun_out/r2t/c3.err
  grep "gemm check" gpurun_out/r2t/c3.err | head -5
done
