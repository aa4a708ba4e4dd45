cd $GRAFT_REPO_ROOT
timeout 600 python tools/spmv_time.py --config c5 > gpurun_out/r2i_spmv.log 2>&1
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 > gpurun_out/r2i_iter.log 2>&1
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 >> gpurun_out/r2i_iter.log 2>&1
cat gpurun_out/r2i_spmv.log gpurun_out/r2i_iter.log
timeout 1500 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_solvers.py tests/test_gpu_kernels.py tests/test_gpu_generation.py tests/test_gpu_ilutp.py -x -q > gpurun_out/r2i_pytest.log 2>&1
tail -2 gpurun_out/r2i_pytest.log
