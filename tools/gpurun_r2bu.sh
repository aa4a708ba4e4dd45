cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_step_timeline.py > gpurun_out/r2bu_timeline.jsonl 2> gpurun_out/r2bu_err.log
cat gpurun_out/r2bu_timeline.jsonl; tail -5 gpurun_out/r2bu_err.log
