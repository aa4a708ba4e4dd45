# round-end evidence: full bench line (default args) and the bench's ncu launch list
set -x
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo BENCH_EXIT $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-synthetic > gpurun_out/ncu_launch_final.log 2>&1; echo NCU $?
