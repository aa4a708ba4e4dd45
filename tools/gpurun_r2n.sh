cd $GRAFT_REPO_ROOT
for v in 0 3 1 0 3; do
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune phase_variant=$v >> gpurun_out/r2n_iter.log 2>&1
done
cat gpurun_out/r2n_iter.log
timeout 900 python -m pytest tests/test_gpu_record.py tests/test_gpu_solvers.py -x -q > gpurun_out/r2n_pytest.log 2>&1
tail -2 gpurun_out/r2n_pytest.log
