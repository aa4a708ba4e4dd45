cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_step_timeline.py --pageable > gpurun_out/r2bw_timeline.jsonl 2> gpurun_out/r2bw_err.log
tail -1 gpurun_out/r2bw_timeline.jsonl; tail -5 gpurun_out/r2bw_err.log
