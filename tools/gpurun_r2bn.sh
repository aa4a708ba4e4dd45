cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -m gpu -q -rf -x > gpurun_out/r2bn_pytest.log 2>&1; tail -4 gpurun_out/r2bn_pytest.log
rm -f gpurun_out/r2bn_*.jsonl
timeout 600 python tools/spmv_time.py --config c5 >> gpurun_out/r2bn_spmv.jsonl 2>gpurun_out/r2bn_err.log
cat gpurun_out/r2bn_spmv.jsonl | cut -c1-200
timeout 900 python tools/ab_iter.py --config c5 --knob value_coding --values 0 1 --rounds 3 > gpurun_out/r2bn_ab.jsonl 2>>gpurun_out/r2bn_err.log; cat gpurun_out/r2bn_ab.jsonl
tail -3 gpurun_out/r2bn_err.log
