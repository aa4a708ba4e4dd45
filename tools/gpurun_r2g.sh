cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_ilutp.py -x -q -s > gpurun_out/r2g_ilutp.log 2>&1
tail -3 gpurun_out/r2g_ilutp.log
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 > gpurun_out/r2g_iter.log 2>&1
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_solvers.py -x -q > gpurun_out/r2g_pytest.log 2>&1
tail -2 gpurun_out/r2g_pytest.log; cat gpurun_out/r2g_iter.log
