cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
echo "bench rc=$?"
CMD="python tools/profile_iter.py --config c5 --solves 1 --max-itn 3"
$CMD > gpurun_out/r2z_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2z_launches.csv $CMD > gpurun_out/r2z_ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_iter_spmv|k_phase<16, 4|k_proj_dot" -s 1 -c 4 -o gpurun_out/r2z_c5_iter $CMD > gpurun_out/r2z_ncu2.log 2>&1
echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_spmv -s 2 -c 1 --csv --log-file gpurun_out/r2z_c4_spmv_l2.csv python tools/spmv_time.py --config c4 --reps 2 > gpurun_out/r2z_ncu3.log 2>&1
echo "ncu3 rc=$?"
