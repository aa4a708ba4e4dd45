cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_ilutp.py -x -q -s > gpurun_out/r2f_ilutp.log 2>&1
tail -3 gpurun_out/r2f_ilutp.log
timeout 1500 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_record.py tests/test_gpu_interop.py -q -s > gpurun_out/r2f_parity.log 2>&1
tail -3 gpurun_out/r2f_parity.log
