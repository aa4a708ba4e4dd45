for v in 0 1 2 3; do echo "PF=$v"; KRB_PF=$v python tools/iter_time.py --config c2 c1 2>&1 | tail -2 | cut -c1-200; done
KRB_PF=2 KRB_PHASE_PROF=1 python tools/iter_time.py --config c2 --phases 2>&1 | tail -1
KRB_PF=3 KRB_PHASE_PROF=1 python tools/iter_time.py --config c2 --phases 2>&1 | tail -1
