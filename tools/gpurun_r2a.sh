set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=memory.used --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_pytest1.log
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
tail -5 gpurun_out/r2_bench_c5.err
