cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q -k "recaptured or large_n" > gpurun_out/r2l_pytest.log 2>&1
tail -2 gpurun_out/r2l_pytest.log
( time timeout 1750 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err ) 2> gpurun_out/r2l_bench.time
tail -3 gpurun_out/r2l_bench.err; cat gpurun_out/r2l_bench.time
