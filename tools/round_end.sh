# round-end measurement set (one box): GPU tests, smoke, every bench workload, the reference arm,
# and the c1 launch list (ncu, after the plain run exited 0)
set -x
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/re_pytest.log 2>&1; tail -2 gpurun_out/re_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; cat gpurun_out/re_smoke.log
timeout 600 python bench.py > gpurun_out/re_c1.json 2> gpurun_out/re_c1.err; tail -1 gpurun_out/re_c1.json
timeout 600 python bench.py > gpurun_out/re_c1b.json 2> gpurun_out/re_c1b.err; tail -1 gpurun_out/re_c1b.json
timeout 600 python bench.py --impl reference > gpurun_out/re_c1_ref.json 2> gpurun_out/re_c1_ref.err; tail -1 gpurun_out/re_c1_ref.json
timeout 600 python bench.py --workload c2 > gpurun_out/re_c2.json 2> gpurun_out/re_c2.err; tail -1 gpurun_out/re_c2.json
timeout 900 python bench.py --workload c3 > gpurun_out/re_c3.json 2> gpurun_out/re_c3.err; tail -1 gpurun_out/re_c3.json
timeout 1200 python bench.py --workload sweep > gpurun_out/re_sweep.json 2> gpurun_out/re_sweep.err; tail -1 gpurun_out/re_sweep.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/re_launches_c1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/re_ncu.log 2>&1; echo ncu rc $?
