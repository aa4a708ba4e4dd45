cd $GRAFT_REPO_ROOT
for v in 0 2 0 2; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune tdot_variant=$v >> gpurun_out/r2q_iter.log 2>&1; done
cat gpurun_out/r2q_iter.log
timeout 900 python tools/iter_time.py --config c3 c4 --max-itn 60 >> gpurun_out/r2q_iter34.log 2>&1; cat gpurun_out/r2q_iter34.log
timeout 1800 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_generation.py -q -x > gpurun_out/r2q_pytest.log 2>&1
tail -3 gpurun_out/r2q_pytest.log
