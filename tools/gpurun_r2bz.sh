cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_step_timeline.py --pageable > gpurun_out/r2bz_timeline_pageable.jsonl 2> gpurun_out/r2bz_err.log
tail -1 gpurun_out/r2bz_timeline_pageable.jsonl; tail -3 gpurun_out/r2bz_err.log
timeout 1200 python tools/e2e_step_timeline.py > gpurun_out/r2bz_timeline_pinned.jsonl 2>> gpurun_out/r2bz_err.log
tail -1 gpurun_out/r2bz_timeline_pinned.jsonl; tail -3 gpurun_out/r2bz_err.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "interop or sequence or policy or generation or kernels" > gpurun_out/r2bz_pytest.log 2>&1; tail -3 gpurun_out/r2bz_pytest.log
