python -m pytest tests/test_gpu_solvers.py -q -x 2>&1 | tail -2
KRB_GRAPH_MODE=2 python tools/profile_iter.py --config c2 --solves 1 && \
KRB_GRAPH_MODE=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_persist2 -c 1 -o gpurun_out/persist2_c2 -f python tools/profile_iter.py --config c2 --solves 1 > gpurun_out/ncu_v2.log 2>&1; tail -2 gpurun_out/ncu_v2.log
