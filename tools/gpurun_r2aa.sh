cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_generation.py tests/test_gpu_solvers.py tests/test_gpu_ilutp.py tests/test_gpu_interop.py tests/test_gpu_batch.py -q -x > gpurun_out/r2aa_pytest.log 2>&1; tail -3 gpurun_out/r2aa_pytest.log
timeout 1200 python tools/c5_step_profile.py --config c5 --systems 3 > gpurun_out/r2aa_step.log 2>&1; grep -v Warn gpurun_out/r2aa_step.log | head -30
