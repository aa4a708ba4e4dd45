cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4 5 0 2; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune spmv_variant=$v > /tmp/o.txt 2>&1; echo "spmv_variant=$v $(cat /tmp/o.txt)" >> gpurun_out/r2ae_iter.log; done
cat gpurun_out/r2ae_iter.log
