cd $GRAFT_REPO_ROOT
timeout 1700 python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
tail -3 gpurun_out/r2_bench_c5.err
