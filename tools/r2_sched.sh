# configs[3] scheduling knobs (1 timed step each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s
for v in "HB_SUBSTREAMS=4" "HB_SUBSTREAMS=6" "HB_SUBSTREAMS=8" "HB_SUBSTREAMS=6 HB_MAX_BIG=4" "HB_SUBSTREAMS=4 HB_CRIT_SHARE=0.5" "HB_SUBSTREAMS=6 HB_BACK_STREAMS=2"; do
  env $v timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2s/c3.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r2s/c3.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity']['equal'], d['parity']['checked_vs_oracle'])"
done
