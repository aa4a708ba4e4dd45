cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -rf > gpurun_out/r2bc_pytest.log 2>&1; tail -5 gpurun_out/r2bc_pytest.log
for t in "" "--transpose"; do
timeout 600 python tools/spmv_time.py --config c5 $t >> gpurun_out/r2bc_spmv.jsonl 2>gpurun_out/r2bc_err.log
timeout 600 python tools/spmv_time.py --config c5 $t --tune value_coding=0 >> gpurun_out/r2bc_spmv.jsonl 2>>gpurun_out/r2bc_err.log
done
cat gpurun_out/r2bc_spmv.jsonl
timeout 900 python tools/ab_iter.py --config c5 --knob value_coding --values 0 1 --rounds 3 > gpurun_out/r2bc_ab.jsonl 2>>gpurun_out/r2bc_err.log; cat gpurun_out/r2bc_ab.jsonl
timeout 600 python tools/spmm_time.py --config c5 >> gpurun_out/r2bc_spmm.jsonl 2>>gpurun_out/r2bc_err.log
timeout 600 python tools/spmm_time.py --config c5 --tune value_coding=0 >> gpurun_out/r2bc_spmm.jsonl 2>>gpurun_out/r2bc_err.log
cat gpurun_out/r2bc_spmm.jsonl; tail -5 gpurun_out/r2bc_err.log
