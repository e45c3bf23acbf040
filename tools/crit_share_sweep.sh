run() { env $1 timeout 200 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/sch_$2.json 2>&1;
        python -c "import json,sys; d=json.loads(open('gpurun_out/sch_$2.json').read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
for rep in 1 2; do
run "HB_CRIT_SHARE=0.25" c25
run "HB_CRIT_SHARE=0.3" c30
run "HB_CRIT_SHARE=0.35" c35
run "HB_CRIT_SHARE=0.4" c40
run "HB_CRIT_SHARE=0.5" c50
done
