cd $GRAFT_REPO_ROOT
timeout 1500 python tools/ab_iter.py --config c5 --knob spmv_prefetch_mb --values 3 4 6 8 12 --rounds 4 >> gpurun_out/r2al_ab.log 2>&1
timeout 1500 python tools/ab_iter.py --config c5 --knob phase_pf_rows --values 0 1 2 --rounds 4 >> gpurun_out/r2al_ab.log 2>&1
cat gpurun_out/r2al_ab.log
