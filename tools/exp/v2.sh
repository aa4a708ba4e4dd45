python tools/iter_time.py --config c1 c2 2>&1 | tail -2
KRB_PHASE_PROF=1 python tools/iter_time.py --config c2 --phases 2>&1 | tail -1
