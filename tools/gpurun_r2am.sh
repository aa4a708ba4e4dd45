cd $GRAFT_REPO_ROOT
timeout 900 python tools/iter_time.py --config c2 --phases >> gpurun_out/r2am_phases.log 2>&1
timeout 900 python tools/iter_time.py --config c2 --k 0 --phases >> gpurun_out/r2am_phases.log 2>&1
timeout 900 python tools/iter_time.py --config c2 c1 --max-itn 100 >> gpurun_out/r2am_phases.log 2>&1
cat gpurun_out/r2am_phases.log
