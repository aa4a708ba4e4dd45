cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rf > gpurun_out/r2be_pytest.log 2>&1; tail -5 gpurun_out/r2be_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_dict" -s 3 -c 1 -o gpurun_out/r2be_c5_spmv_vc python tools/spmv_time.py --config c5 --reps 2 > gpurun_out/r2be_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2be_ncu.log
