# persist0: grid = #SMs (default) vs one CTA per two canonical blocks (KRB_P0_GRID=half)
for m in full half full half; do
  KRB_P0_GRID=$m timeout 120 python tools/iter_time.py --config c2 --k 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grid=$m', d['us_per_it'])"
done
