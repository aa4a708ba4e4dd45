cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_phases.py --config c5 --systems 3 > gpurun_out/r2bq_e2e_phases.jsonl 2> gpurun_out/r2bq_err.log
cat gpurun_out/r2bq_e2e_phases.jsonl; tail -3 gpurun_out/r2bq_err.log
