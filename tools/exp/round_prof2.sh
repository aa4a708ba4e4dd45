set -x
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH_EXIT $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-synthetic > gpurun_out/ncu_launch.log 2>&1; echo NCU1 $?
KRB_GRAPH_MODE=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_persist0 -c 1 -o gpurun_out/persist0_c2 -f python tools/profile_iter.py --config c2 --solves 1 --k 0 > gpurun_out/ncu_p0.log 2>&1; echo NCU2 $?
tail -3 gpurun_out/ncu_p0.log
