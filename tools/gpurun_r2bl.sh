cd $GRAFT_REPO_ROOT
rm -f gpurun_out/r2bl_*.jsonl
timeout 600 python tools/spmv_time.py --config c5 >> gpurun_out/r2bl_spmv.jsonl 2>gpurun_out/r2bl_err.log
timeout 600 python tools/spmv_time.py --config c5 --transpose >> gpurun_out/r2bl_spmv.jsonl 2>>gpurun_out/r2bl_err.log
timeout 600 python tools/spmv_time.py --config c2 >> gpurun_out/r2bl_spmv.jsonl 2>>gpurun_out/r2bl_err.log
timeout 600 python tools/spmv_time.py --config c1 >> gpurun_out/r2bl_spmv.jsonl 2>>gpurun_out/r2bl_err.log
cat gpurun_out/r2bl_spmv.jsonl | cut -c1-200
timeout 900 python tools/ab_iter.py --config c5 --knob value_coding --values 0 1 2 --rounds 3 > gpurun_out/r2bl_ab.jsonl 2>>gpurun_out/r2bl_err.log; cat gpurun_out/r2bl_ab.jsonl
timeout 900 python tools/ab_iter.py --config c3 --knob value_coding --values 0 1 --rounds 3 >> gpurun_out/r2bl_ab.jsonl 2>>gpurun_out/r2bl_err.log; tail -1 gpurun_out/r2bl_ab.jsonl
tail -3 gpurun_out/r2bl_err.log
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/r2bl_pytest.log 2>&1; tail -5 gpurun_out/r2bl_pytest.log
