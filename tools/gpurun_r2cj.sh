cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py -m gpu -q > gpurun_out/r2cj_pytest.log 2>&1; tail -2 gpurun_out/r2cj_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tools/spmv_time.py --config c5 2>/dev/null | cut -c1-140
