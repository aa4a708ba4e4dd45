cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab_iter.py --config c5 --knob spmv_variant --values 0 1 2 3 4 --rounds 4 >> gpurun_out/r2ai_ab.log 2>&1
cat gpurun_out/r2ai_ab.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x > gpurun_out/r2ai_pytest.log 2>&1; tail -2 gpurun_out/r2ai_pytest.log
