# c1 scheduling knobs (sub-streams, back-of-queue streams, critical-stream SM share); 8 steps each
run() { env $1 timeout 200 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/sch_$2.json 2>&1;
        python -c "import json,sys; d=json.loads(open('gpurun_out/sch_$2.json').read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
run "HB_SUBSTREAMS=4" base4
run "HB_SUBSTREAMS=4 HB_CRIT_SHARE=0.35" s4c35
run "HB_SUBSTREAMS=4 HB_CRIT_SHARE=0.65" s4c65
run "HB_SUBSTREAMS=3" s3
run "HB_SUBSTREAMS=3 HB_CRIT_SHARE=0.4" s3c40
run "HB_SUBSTREAMS=5" s5
run "HB_SUBSTREAMS=5 HB_CRIT_SHARE=0.35" s5c35
run "HB_SUBSTREAMS=4 HB_BACK_STREAMS=1" b41
run "HB_SUBSTREAMS=6 HB_BACK_STREAMS=2 HB_CRIT_SHARE=0.35" b62c
run "HB_SUBSTREAMS=4" base4b
