cd $GRAFT_REPO_ROOT
timeout 1200 python tools/ab_iter.py --config c5 --knob phase_pf_rows --values 0 1 2 4 --rounds 4 >> gpurun_out/r2af_ab.log 2>&1
timeout 1200 python tools/ab_iter.py --config c5 --knob spmv_variant --values 0 1 --rounds 4 >> gpurun_out/r2af_ab.log 2>&1
timeout 900 python tools/ab_iter.py --config c3 --system 1 --knob phase_pf_rows --values 0 1 2 4 --rounds 4 >> gpurun_out/r2af_ab.log 2>&1
cat gpurun_out/r2af_ab.log
timeout 600 python tools/spmv_time.py --config c5 >> gpurun_out/r2af_spmv.log 2>&1; cat gpurun_out/r2af_spmv.log
