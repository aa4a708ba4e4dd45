cd $GRAFT_REPO_ROOT
rm -f gpurun_out/r2cc_spmv.jsonl
for b in 256 128 512 1024 256; do
timeout 600 python tools/spmv_time.py --config c5 --tune spmv_block=$b >> gpurun_out/r2cc_spmv.jsonl 2>gpurun_out/r2cc_err.log
done
cut -c1-140 gpurun_out/r2cc_spmv.jsonl; grep -o '"tune": .*' gpurun_out/r2cc_spmv.jsonl; tail -2 gpurun_out/r2cc_err.log
