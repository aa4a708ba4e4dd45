cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_persistent.py -k "staged or large_n" tests/test_gpu_record.py tests/test_gpu_interop.py -x -q > gpurun_out/r2d_pytest.log 2>&1
tail -3 gpurun_out/r2d_pytest.log
timeout 600 python tools/spmv_time.py --config c5 > gpurun_out/r2d_spmv.log 2>&1
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 > gpurun_out/r2d_iter.log 2>&1
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune corr_staged=0 >> gpurun_out/r2d_iter.log 2>&1
cat gpurun_out/r2d_spmv.log gpurun_out/r2d_iter.log | tail -5
