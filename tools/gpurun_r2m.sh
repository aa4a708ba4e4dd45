cd $GRAFT_REPO_ROOT
CMD="python tools/profile_iter.py --config c5 --solves 1 --max-itn 3"
$CMD > gpurun_out/r2m_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_launches.csv $CMD > gpurun_out/r2m_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_iter_spmv|k_proj_dot|k_phase" -s 2 -c 9 -o gpurun_out/r2m_c5_iter $CMD > gpurun_out/r2m_ncu2.log 2>&1
echo rc=$?
tail -3 gpurun_out/r2m_ncu2.log
