cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py -m gpu -q -rf > gpurun_out/r2bv_pytest.log 2>&1; tail -4 gpurun_out/r2bv_pytest.log
