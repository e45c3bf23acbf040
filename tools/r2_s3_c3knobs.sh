# configs[3] (bench default) against the shared-queue knobs: 1 warm-up + 2 timed steps each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s3
run() {
  name=$1; shift
  env "$@" timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2s3/knob_$name.json 2> gpurun_out/r2s3/knob_$name.err
  python -c "import json; d=json.loads(open('gpurun_out/r2s3/knob_$name.json').read().strip().splitlines()[-1]); print('$name', d['ms_per_step'], 'parity', d['parity']['checked_vs_oracle'], d['parity']['equal'])"
}
run default HB_SUBSTREAMS=4
run big2 HB_MAX_BIG=2
run big4 HB_MAX_BIG=4
run s5 HB_SUBSTREAMS=5
run s6 HB_SUBSTREAMS=6
run s6big4 HB_SUBSTREAMS=6 HB_MAX_BIG=4
run s3 HB_SUBSTREAMS=3
run crit50 HB_CRIT_SHARE=0.5
run crit25 HB_CRIT_SHARE=0.25
run back1 HB_BACK_STREAMS=1
run s5back1 HB_SUBSTREAMS=5 HB_BACK_STREAMS=1
run nopri HB_NO_PRIORITY=1
