# certified golden records of sweep problems outside configs[3] on the GPU box's 16 host cores
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/boxcpu3
export OPENBLAS_NUM_THREADS=$(nproc)
timeout 2150 python tests/golden/make_baseline_ranks.py --certified --skip-c3 --max-cost 6000 --out gpurun_out/boxcpu3/golden_box.json --deadline 2100 > gpurun_out/boxcpu3/golden.log 2>&1
tail -12 gpurun_out/boxcpu3/golden.log | cut -c1-200
