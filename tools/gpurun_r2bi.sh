cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_dict" -s 3 -c 1 -o gpurun_out/r2bi_c5_spmv_dia3 python tools/spmv_time.py --config c5 --reps 2 > gpurun_out/r2bi_ncu.log 2>&1
echo rc=$?
