python -m pytest tests/test_gpu_persistent.py -q -x 2>&1 | tail -2
python tools/iter_time.py --config c2 c1 --both 2>&1 | tail -4 | cut -c1-220
KRB_PHASE_PROF=1 python tools/iter_time.py --config c2 --phases 2>&1 | tail -1
