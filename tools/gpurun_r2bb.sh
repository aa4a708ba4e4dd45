cd $GRAFT_REPO_ROOT
S=$(date +%s); timeout 2400 python bench.py > gpurun_out/r2bb_bench.json 2> gpurun_out/r2bb_bench.err; echo "bench rc=$? $(( $(date +%s) - S )) s"
S=$(date +%s); timeout 1800 python bench.py --impl reference > gpurun_out/r2bb_ref.json 2> gpurun_out/r2bb_ref.err; echo "ref rc=$? $(( $(date +%s) - S )) s"
