cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_generation.py tests/test_gpu_fullsize.py tests/test_gpu_ilutp.py -q -x > gpurun_out/r2aj_pytest.log 2>&1; tail -2 gpurun_out/r2aj_pytest.log
timeout 1800 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2aj_bench.json 2> gpurun_out/r2aj_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2aj_bench.json').read().strip().splitlines()[-1]); print(d['value'], d.get('full_policy'))"
