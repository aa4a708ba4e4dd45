cd $GRAFT_REPO_ROOT
for cfg in "spmm_panel=1" "spmm_panel=0" "spmm_panel=1"; do timeout 600 python tools/spmm_time.py --config c5 --ncols 30 --tune $cfg >> gpurun_out/r2y_spmm.log 2>&1; done
cat gpurun_out/r2y_spmm.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_generation.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2y_pytest.log 2>&1; tail -2 gpurun_out/r2y_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -s > gpurun_out/r2y_parity.log 2>&1; tail -2 gpurun_out/r2y_parity.log
timeout 1200 python tools/c5_step_profile.py --config c5 --systems 2 > gpurun_out/r2y_step.log 2>&1; grep -v Warn gpurun_out/r2y_step.log | head -24
