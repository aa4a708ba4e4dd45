cd $GRAFT_REPO_ROOT
for f in 2 4 4; do timeout 300 python tools/spmv_time.py --config c5 --fmt $f >> gpurun_out/r2r_spmv.log 2>&1; done
cat gpurun_out/r2r_spmv.log
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 > gpurun_out/r2r_iter.log 2>&1; cat gpurun_out/r2r_iter.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_dict -s 3 -c 1 -o gpurun_out/r2r_spmv_dict python tools/spmv_time.py --config c5 --fmt 4 --reps 2 > gpurun_out/r2r_ncu.log 2>&1
echo ncu rc=$?
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x > gpurun_out/r2r_pytest.log 2>&1; tail -2 gpurun_out/r2r_pytest.log
