cd $GRAFT_REPO_ROOT
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 > gpurun_out/r2h_iter.log 2>&1
cat gpurun_out/r2h_iter.log
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_solvers.py tests/test_gpu_kernels.py -x -q > gpurun_out/r2h_pytest.log 2>&1
tail -2 gpurun_out/r2h_pytest.log
timeout 1500 python tools/c4_convergence.py --max-itn 5000 > gpurun_out/r2h_c4.log 2>&1
cat gpurun_out/r2h_c4.log
