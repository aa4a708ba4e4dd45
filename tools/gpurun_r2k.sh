cd $GRAFT_REPO_ROOT
timeout 900 python tools/iter_time.py --config c5 --max-itn 60 > gpurun_out/r2k_iter.log 2>&1
cat gpurun_out/r2k_iter.log
( time timeout 1750 python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err ) 2> gpurun_out/r2k_bench.time
tail -3 gpurun_out/r2k_bench.err; cat gpurun_out/r2k_bench.time
( time timeout 1750 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2k_ref.json 2> gpurun_out/r2k_ref.err ) 2> gpurun_out/r2k_ref.time
tail -3 gpurun_out/r2k_ref.err; cat gpurun_out/r2k_ref.time
