cd $GRAFT_REPO_ROOT
S=$(date +%s); timeout 2400 python bench.py --steps 10 --warmup 3 > gpurun_out/r2cg_bench10.json 2> gpurun_out/r2cg_bench10.err; echo "bench rc=$? $(( $(date +%s) - S )) s"
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/r2cg_bench10.json") if l.startswith("{")][-1])
print(d["value"], d["step_ms"], d["e2e"]["value"], d["e2e"]["steps"], d["e2e_pageable"]["value"], d["roofline"]["frac"], d["clocks"])
PY
