cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ao_build.log 2>&1; echo "build rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/r2ao_pytest.log 2>&1; tail -3 gpurun_out/r2ao_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ao_smoke.log 2>&1; tail -1 gpurun_out/r2ao_smoke.log
/usr/bin/time -v timeout 2400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2ao_bench.json 2> gpurun_out/r2ao_bench.err; echo "bench rc=$?"; grep "Elapsed\|Maximum resident" gpurun_out/r2ao_bench.err
/usr/bin/time -v timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2ao_ref.json 2> gpurun_out/r2ao_ref.err; echo "ref rc=$?"; grep "Elapsed\|Maximum resident" gpurun_out/r2ao_ref.err
