cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solvers.py -m gpu -q -rf -x -k "fused or value_coding" > gpurun_out/r2bt_pytest.log 2>&1; tail -4 gpurun_out/r2bt_pytest.log
timeout 900 python tools/ab_iter.py --config c5 --knob fuse_spmv_dot --values 0 1 --rounds 3 > gpurun_out/r2bt_ab.jsonl 2>gpurun_out/r2bt_err.log; cat gpurun_out/r2bt_ab.jsonl
tail -3 gpurun_out/r2bt_err.log
