# sweep: large problems solo (default) vs on concurrent sub-streams with the small ones
run() { env $1 timeout 900 python bench.py --workload sweep --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/lo_$2.json 2>&1;
        python -c "import json; d=json.loads(open('gpurun_out/lo_$2.json').read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['parity']['equal'], d['parity']['checked_vs_oracle'], d['parity']['statuses_ok'])"; }
run "HB_SMALL_N=70000 HB_SMALL_RANK=1e9 HB_SUBSTREAMS=2 HB_CRIT_SHARE=0.5" all2
run "HB_SMALL_N=70000 HB_SMALL_RANK=1e9 HB_SUBSTREAMS=3" all3
run "HB_SMALL_N=40000 HB_SMALL_RANK=1e9 HB_SUBSTREAMS=4" n40k
