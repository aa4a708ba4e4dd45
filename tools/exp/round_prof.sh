set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --systems 2 > gpurun_out/b_small.json 2>/dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --systems 2 > gpurun_out/ncu_launch.log 2>&1
KRB_GRAPH_MODE=2 python tools/profile_iter.py --config c2 --solves 1 || exit 1
KRB_GRAPH_MODE=2 ncu --set full --import-source on --clock-control none -k regex:k_persist2 -c 1 -o gpurun_out/persist2_c2 -f python tools/profile_iter.py --config c2 --solves 1 > gpurun_out/ncu_v2.log 2>&1
tail -2 gpurun_out/ncu_v2.log
