cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2bs_build.log 2>&1; echo "build rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/r2bs_pytest.log 2>&1; tail -3 gpurun_out/r2bs_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bs_smoke.log 2>&1; tail -1 gpurun_out/r2bs_smoke.log
S=$(date +%s); timeout 2400 python bench.py > gpurun_out/r2bs_bench.json 2> gpurun_out/r2bs_bench.err; echo "bench rc=$? $(( $(date +%s) - S )) s"
S=$(date +%s); timeout 1800 python bench.py --impl reference > gpurun_out/r2bs_ref.json 2> gpurun_out/r2bs_ref.err; echo "ref rc=$? $(( $(date +%s) - S )) s"
S=$(date +%s); timeout 1200 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r2bs_bench_c2.json 2> gpurun_out/r2bs_bench_c2.err; echo "c2 rc=$? $(( $(date +%s) - S )) s"
