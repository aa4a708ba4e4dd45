cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --steps 1 --warmup 1 > gpurun_out/r2cb_bench.json 2> gpurun_out/r2cb_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/r2cb_bench.json") if l.startswith("{")][-1])
print(d["value"], d["e2e"]["value"], d["parity"])
PY
tail -3 gpurun_out/r2cb_bench.err
