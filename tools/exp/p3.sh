python -m pytest tests/test_gpu_persistent.py -q -x 2>&1 | tail -2
for c in c3 c5; do
KRB_GRAPH_MODE=2 python tools/iter_time.py --config $c --both 2>&1 | cut -c1-200
KRB_GRAPH_MODE=1 python tools/iter_time.py --config $c --both 2>&1 | cut -c1-200
done
