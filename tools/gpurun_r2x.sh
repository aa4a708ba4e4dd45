cd $GRAFT_REPO_ROOT
for cfg in "tdot_variant=0" "tdot_variant=4" "tdot_variant=0" "tdot_variant=4"; do timeout 900 python tools/iter_time.py --config c3 --system 1 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2x_iter.log; done
timeout 900 python tools/iter_time.py --config c5 c2 --max-itn 60 > /tmp/o.txt 2>&1; cat /tmp/o.txt >> gpurun_out/r2x_iter.log
cat gpurun_out/r2x_iter.log
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/r2x_pytest.log 2>&1
tail -8 gpurun_out/r2x_pytest.log
