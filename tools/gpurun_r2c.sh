cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_record.py tests/test_gpu_interop.py -x -q -s > gpurun_out/r2_pytest_new.log 2>&1
tail -3 gpurun_out/r2_pytest_new.log
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench_c5b.json 2> gpurun_out/r2_bench_c5b.err
tail -3 gpurun_out/r2_bench_c5b.err
timeout 900 python tools/e2e_phases.py --systems 3 > gpurun_out/r2_e2e_phases.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_all.log 2>&1
tail -3 gpurun_out/r2_pytest_all.log
