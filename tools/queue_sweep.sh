# sweep workload: sub-stream count, big-problem cap and critical-stream share
run() { env $1 timeout 900 python bench.py --workload sweep --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/qs_$2.json 2>&1;
        python -c "import json; d=json.loads(open('gpurun_out/qs_$2.json').read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['parity']['equal'], d['parity']['statuses_ok'])"; }
run "HB_MAX_BIG=2" b2
run "HB_CRIT_SHARE=0.5" c50
run "HB_SUBSTREAMS=5" s5
run "HB_MAX_BIG=3" b3
