cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rf -x > gpurun_out/r2bf_pytest.log 2>&1; tail -5 gpurun_out/r2bf_pytest.log
rm -f gpurun_out/r2bf_*.jsonl
for t in "" "--transpose"; do
timeout 600 python tools/spmv_time.py --config c5 $t >> gpurun_out/r2bf_spmv.jsonl 2>gpurun_out/r2bf_err.log
timeout 600 python tools/spmv_time.py --config c5 $t --tune value_coding=2 >> gpurun_out/r2bf_spmv.jsonl 2>>gpurun_out/r2bf_err.log
done
timeout 600 python tools/spmv_time.py --config c2 >> gpurun_out/r2bf_spmv.jsonl 2>>gpurun_out/r2bf_err.log
timeout 600 python tools/spmv_time.py --config c2 --tune value_coding=0 >> gpurun_out/r2bf_spmv.jsonl 2>>gpurun_out/r2bf_err.log
cat gpurun_out/r2bf_spmv.jsonl
timeout 900 python tools/ab_iter.py --config c5 --knob value_coding --values 0 1 2 --rounds 3 > gpurun_out/r2bf_ab.jsonl 2>>gpurun_out/r2bf_err.log; cat gpurun_out/r2bf_ab.jsonl
tail -5 gpurun_out/r2bf_err.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_dict" -s 3 -c 1 -o gpurun_out/r2bf_c5_spmv_dia python tools/spmv_time.py --config c5 --reps 2 > gpurun_out/r2bf_ncu.log 2>&1
