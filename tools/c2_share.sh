# c2 spread: critical-stream share 0.25 (equal caps) vs the default 0.35, two runs each
run() { env $1 timeout 300 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2s_$2.json 2>&1;
        python -c "import json; d=json.loads(open('gpurun_out/c2s_$2.json').read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['parity']['equal'], d['parity']['statuses_ok'])"; }
run "HB_CRIT_SHARE=0.25" a1
run "HB_CRIT_SHARE=0.35" b1
run "HB_CRIT_SHARE=0.25" a2
run "HB_CRIT_SHARE=0.35" b2
run "HB_CRIT_SHARE=0.25 HB_SUBSTREAMS=5 HB_MAX_BIG=4" c1
run "HB_CRIT_SHARE=0.35 HB_SUBSTREAMS=5 HB_MAX_BIG=4" d1
