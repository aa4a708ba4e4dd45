# persist0: phase A operands prefetched across the scalar barrier (KRB_P0_PRE=1) vs not (0)
timeout 300 python -m pytest tests/test_gpu_persist0.py -x -q 2>&1 | tail -1
for m in 0 1 0 1; do
  KRB_P0_PRE=$m timeout 120 python tools/iter_time.py --config c2 --k 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pre=$m', d['us_per_it'])"
done
