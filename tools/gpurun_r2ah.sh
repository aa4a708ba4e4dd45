cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_generation.py tests/test_gpu_interop.py tests/test_gpu_kernels.py -q -x > gpurun_out/r2ah_pytest.log 2>&1; tail -2 gpurun_out/r2ah_pytest.log
timeout 1800 python bench.py --steps 3 --warmup 3 --no-policy --no-cpu-baseline > gpurun_out/r2ah_bench.json 2> gpurun_out/r2ah_bench.err; echo "bench rc=$?"
