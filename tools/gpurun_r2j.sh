cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune phase_variant=$v >> gpurun_out/r2j_iter.log 2>&1
done
cat gpurun_out/r2j_iter.log
