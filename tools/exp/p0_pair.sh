# persist0: interleaved owned rows (KRB_P0_PAIR=1, default) vs one by one (0)
timeout 300 python -m pytest tests/test_gpu_persist0.py -x -q 2>&1 | tail -1
for m in 0 1 0 1; do
  KRB_P0_PAIR=$m timeout 120 python tools/iter_time.py --config c2 --k 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pair=$m', d['us_per_it'])"
done
KRB_P0_PAIR=1 timeout 120 python tools/exp/p0cta.py c2 0,108 2>/dev/null
