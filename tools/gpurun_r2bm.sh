cd $GRAFT_REPO_ROOT
S=$(date +%s); timeout 2400 python bench.py > gpurun_out/r2bm_bench.json 2> gpurun_out/r2bm_bench.err; echo "bench rc=$? $(( $(date +%s) - S )) s"
CMD="python tools/profile_iter.py --config c5 --solves 1 --max-itn 3"
$CMD > gpurun_out/r2bm_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bm_launches.csv $CMD > gpurun_out/r2bm_ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_iter_spmv|k_phase|k_proj_dot" -s 9 -c 9 -o gpurun_out/r2bm_c5_iter $CMD > gpurun_out/r2bm_ncu2.log 2>&1
echo "ncu rc=$?"
S=$(date +%s); timeout 1800 python bench.py --impl reference > gpurun_out/r2bm_ref.json 2> gpurun_out/r2bm_ref.err; echo "ref rc=$? $(( $(date +%s) - S )) s"
