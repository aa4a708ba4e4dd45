cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_step_timeline.py > gpurun_out/r2ce_timeline_pinned.jsonl 2> gpurun_out/r2ce_err.log
python - <<'PY'
import json
for l in open("gpurun_out/r2ce_timeline_pinned.jsonl"):
    d=json.loads(l); print(d["rep"], d["total_s"], [(r["sys"], r.get("adopt_prefetch"), r.get("device_matrix")) for r in d["log"][1:3]])
PY
timeout 1200 python tools/e2e_step_timeline.py --pageable > gpurun_out/r2ce_timeline_pageable.jsonl 2>> gpurun_out/r2ce_err.log
python - <<'PY'
import json
for l in open("gpurun_out/r2ce_timeline_pageable.jsonl"):
    d=json.loads(l); print(d["rep"], d["total_s"], [(r["sys"], r.get("adopt_prefetch"), r.get("device_matrix")) for r in d["log"][1:4]])
PY
timeout 900 python -m pytest tests -m gpu -q -x -k "sequence or policy or interop or generation" > gpurun_out/r2ce_pytest.log 2>&1; tail -2 gpurun_out/r2ce_pytest.log
