# CPU-only work on the GPU box's host cores (more cores and memory than the build container):
# the independent CPU check of the paper's 3-D N = 64000 values, then certified golden records of
# the sweep problems outside configs[3] (the build container works on configs[3] meanwhile).
# Outputs under gpurun_out/boxcpu/ (merged into tests/golden/ afterwards).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/boxcpu
nproc; free -g | head -2
timeout 1500 python -m pytest tests/test_gpu_rank.py -q -m gpu -x -k 'two_workers or bad_arguments or fp_band or tma_update' > gpurun_out/boxcpu/pytest_rest.log 2>&1; tail -3 gpurun_out/boxcpu/pytest_rest.log
export OPENBLAS_NUM_THREADS=$(nproc)
( while true; do cp -f tests/golden/paper_check_n64000.json gpurun_out/boxcpu/ 2>/dev/null; sleep 30; done ) &
CP=$!
timeout ${PAPER_S:-3600} python tests/golden/make_paper_check.py > gpurun_out/boxcpu/paper_check.log 2>&1
cp -f tests/golden/paper_check_n64000.json gpurun_out/boxcpu/ 2>/dev/null
tail -6 gpurun_out/boxcpu/paper_check.log | cut -c1-300
timeout ${GOLD_S:-3000} python tests/golden/make_baseline_ranks.py --certified --skip-c3 --max-cost 6000 --out gpurun_out/boxcpu/golden_box.json --deadline ${GOLD_S:-3000} > gpurun_out/boxcpu/golden.log 2>&1
tail -12 gpurun_out/boxcpu/golden.log | cut -c1-200
kill $CP
