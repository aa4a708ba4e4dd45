cd $GRAFT_REPO_ROOT
timeout 1500 python tools/policy_profile.py --config c5 --top 40 > gpurun_out/r2ak_policy.log 2>&1; grep -v Warn gpurun_out/r2ak_policy.log | head -50
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "spmv" > gpurun_out/r2ak_pytest.log 2>&1; tail -2 gpurun_out/r2ak_pytest.log
