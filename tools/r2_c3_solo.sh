cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
HB_TIMELINE=1 timeout 900 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline --details gpurun_out/r2a/c3_details.json > gpurun_out/r2a/c3.json 2> gpurun_out/r2a/c3.err
tail -c 1500 gpurun_out/r2a/c3.json
timeout 600 python tools/solo.py 4 3 one_over_r 65536 1 1e-12 > gpurun_out/r2a/solo_4d3_inv.log 2>&1
timeout 600 python tools/solo.py 4 3 exp_neg_r 65536 1 > gpurun_out/r2a/solo_4d3_exp.log 2>&1
cat gpurun_out/r2a/solo_*.log
