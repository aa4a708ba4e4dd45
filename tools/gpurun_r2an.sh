cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_iter.py --config c2 --knob persist_dict --values 0 1 --rounds 6 --max-itn 200 >> gpurun_out/r2an_ab.log 2>&1
timeout 900 python tools/ab_iter.py --config c2 --system 5 --knob persist_dict --values 0 1 --rounds 6 --max-itn 200 >> gpurun_out/r2an_ab.log 2>&1
cat gpurun_out/r2an_ab.log
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_persistent.py tests/test_gpu_edge.py -q -x > gpurun_out/r2an_pytest.log 2>&1; tail -2 gpurun_out/r2an_pytest.log
