cd $GRAFT_REPO_ROOT
for cfg in "phase_prefetch=0" "phase_prefetch=1" "phase_prefetch=2" "phase_prefetch=0" "phase_prefetch=1" "phase_prefetch=2"; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2w_iter.log; done
cat gpurun_out/r2w_iter.log
for cfg in "spmv_prefetch_mb=0" "spmv_prefetch_mb=6" "spmv_prefetch_mb=6 phase_prefetch=1" "spmv_prefetch_mb=6 phase_prefetch=2"; do timeout 900 python tools/iter_time.py --config c4 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2w_iter4.log;
timeout 900 python tools/iter_time.py --config c3 --system 1 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2w_iter4.log; done
cat gpurun_out/r2w_iter4.log
