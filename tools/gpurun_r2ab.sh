cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -x > gpurun_out/r2ab_pytest.log 2>&1; tail -2 gpurun_out/r2ab_pytest.log
for cfg in "phase_grid=0" "phase_grid=1" "phase_grid=2" "phase_grid=0" "phase_grid=1" "phase_grid=2"; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2ab_iter.log; done
for cfg in "phase_grid=0" "phase_grid=1" "phase_grid=2"; do timeout 900 python tools/iter_time.py --config c3 --system 1 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2ab_iter.log; done
cat gpurun_out/r2ab_iter.log
timeout 1200 python tools/c5_step_profile.py --config c5 --systems 3 > gpurun_out/r2ab_step.log 2>&1; grep "system\|iterations" gpurun_out/r2ab_step.log
