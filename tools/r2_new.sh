cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2r
timeout 900 python -m pytest tests/test_gpu_hmatrix.py tests/test_gpu_chebyshev.py tests/test_cli.py -q -x > gpurun_out/r2r/pytest_new.log 2>&1; tail -15 gpurun_out/r2r/pytest_new.log
