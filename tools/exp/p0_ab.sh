# persist0 hand-off A/B: flag-polled vs data-polled (C2 k=0) + parity tests
set -x
timeout 300 python -m pytest tests/test_gpu_persist0.py -x -q 2>&1 | tail -2
for m in flags data flags data; do
  KRB_P0_HANDOFF=$m timeout 120 python tools/iter_time.py --config c2 --k 0 2>/dev/null
done
KRB_P0_HANDOFF=data timeout 120 python tools/exp/p0cta.py c2 0,108 2>/dev/null
