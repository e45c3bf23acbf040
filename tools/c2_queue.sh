# c2 (d=3, N up to 32768): big-problem cap and stream count
run() { env $1 timeout 300 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2q_$2.json 2>&1;
        python -c "import json; d=json.loads(open('gpurun_out/c2q_$2.json').read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['parity']['equal'], d['parity']['statuses_ok'])"; }
run "HB_MAX_BIG=3" b3
run "HB_MAX_BIG=4" b4
run "HB_MAX_BIG=6 HB_SUBSTREAMS=6" b6s6
run "HB_MAX_BIG=5 HB_SUBSTREAMS=5" b5s5
run "HB_MAX_BIG=4 HB_SUBSTREAMS=5" b4s5
run "HB_MAX_BIG=3" b3b
