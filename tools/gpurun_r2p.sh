cd $GRAFT_REPO_ROOT
timeout 600 python tools/diag_c1.py c1 > gpurun_out/r2p_diag.log 2>&1; tail -30 gpurun_out/r2p_diag.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "offset_coded or formats" > gpurun_out/r2p_dict_tests.log 2>&1; tail -3 gpurun_out/r2p_dict_tests.log
for f in 2 4 2 4; do timeout 300 python tools/spmv_time.py --config c5 --fmt $f >> gpurun_out/r2p_spmv.log 2>&1; done
timeout 300 python tools/spmv_time.py --config c5 --fmt 4 --transpose >> gpurun_out/r2p_spmv.log 2>&1
timeout 300 python tools/spmv_time.py --config c2 --fmt 2 >> gpurun_out/r2p_spmv.log 2>&1
timeout 300 python tools/spmv_time.py --config c2 --fmt 4 >> gpurun_out/r2p_spmv.log 2>&1
cat gpurun_out/r2p_spmv.log
for f in 2 4; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --fmt $f >> gpurun_out/r2p_iter.log 2>&1; done
cat gpurun_out/r2p_iter.log
timeout 2400 python -m pytest tests -m gpu -q --deselect "tests/test_gpu_parity_full.py::test_full_size_solvers_vs_reference[c1-3]" > gpurun_out/r2p_pytest.log 2>&1
tail -5 gpurun_out/r2p_pytest.log
