# C4 per-kernel launch list (host-loop driver, a few iterations) + one full capture of each SpMV kernel
set -x
export KRB_GRAPH_MODE=0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_iter_spmv|k_proj_dot|k_phase" --launch-skip 30 -c 36 --csv --log-file gpurun_out/c4_launches.csv \
  python tools/profile_iter.py --config c4 --solves 1 > gpurun_out/c4_l.log 2>&1; echo NCU1 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_iter_spmv --launch-skip 4 -c 1 \
  -o gpurun_out/c4_spmv -f python tools/profile_iter.py --config c4 --solves 1 > gpurun_out/c4_f.log 2>&1; echo NCU2 $?
