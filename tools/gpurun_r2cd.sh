cd $GRAFT_REPO_ROOT
CMD="python tools/profile_iter.py --config c5 --solves 1 --max-itn 3"
$CMD > gpurun_out/r2cd_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2cd_launches.csv $CMD > gpurun_out/r2cd_ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_iter_spmv|k_phase|k_proj_dot" -s 9 -c 9 -o gpurun_out/r2cd_c5_iter $CMD > gpurun_out/r2cd_ncu2.log 2>&1
echo "ncu rc=$?"
