cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rf -x > gpurun_out/r2bg_pytest.log 2>&1; tail -5 gpurun_out/r2bg_pytest.log
rm -f gpurun_out/r2bg_*.jsonl
timeout 600 python tools/spmv_time.py --config c5 >> gpurun_out/r2bg_spmv.jsonl 2>gpurun_out/r2bg_err.log
timeout 600 python tools/spmv_time.py --config c5 --tune value_coding=2 >> gpurun_out/r2bg_spmv.jsonl 2>>gpurun_out/r2bg_err.log
cat gpurun_out/r2bg_spmv.jsonl
tail -5 gpurun_out/r2bg_err.log
