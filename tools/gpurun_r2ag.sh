cd $GRAFT_REPO_ROOT
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/r2ag_pytest.log 2>&1; tail -3 gpurun_out/r2ag_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ag_smoke.log 2>&1; tail -1 gpurun_out/r2ag_smoke.log
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/r2ag_bench.json 2> gpurun_out/r2ag_bench.err; echo "bench rc=$?"
