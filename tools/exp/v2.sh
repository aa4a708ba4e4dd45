python -m pytest tests/test_gpu_solvers.py -q -x 2>&1 | tail -2
for v in 1 0; do echo "L2PERSIST=$v"; KRB_L2PERSIST=$v python tools/iter_time.py --config c1 c2 2>&1 | tail -2
KRB_L2PERSIST=$v KRB_PHASE_PROF=1 python tools/iter_time.py --config c2 --phases 2>&1 | tail -1; done
