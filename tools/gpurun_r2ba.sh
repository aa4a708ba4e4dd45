cd $GRAFT_REPO_ROOT
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/r2ba_pytest.log 2>&1; tail -3 gpurun_out/r2ba_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ba_smoke.log 2>&1; tail -1 gpurun_out/r2ba_smoke.log
/usr/bin/time -v timeout 2400 python bench.py > gpurun_out/r2ba_bench.json 2> gpurun_out/r2ba_bench.err; echo "bench rc=$?"; grep "Elapsed\|Maximum resident" gpurun_out/r2ba_bench.err
/usr/bin/time -v timeout 1800 python bench.py --impl reference > gpurun_out/r2ba_ref.json 2> gpurun_out/r2ba_ref.err; echo "ref rc=$?"; grep "Elapsed\|Maximum resident" gpurun_out/r2ba_ref.err
