cd $GRAFT_REPO_ROOT
for cfg in "spmv_prefetch_mb=2" "spmv_prefetch_mb=4" "spmv_prefetch_mb=6" "spmv_prefetch_mb=8" "spmv_prefetch_mb=0" "spmv_prefetch_mb=4" "spmv_prefetch_mb=6"; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2v_iter.log; done
cat gpurun_out/r2v_iter.log
for cfg in "spmv_prefetch_mb=0" "spmv_prefetch_mb=6"; do timeout 900 python tools/iter_time.py --config c3 c2 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2v_iter3.log; done
cat gpurun_out/r2v_iter3.log
timeout 1200 python tools/c5_step_profile.py --config c5 --systems 2 > gpurun_out/r2v_step.log 2>&1; cat gpurun_out/r2v_step.log
