cd $GRAFT_REPO_ROOT
cat > /tmp/sv.py <<'PY'
import sys, subprocess
PY
for v in 0 1 0 1; do timeout 300 python -c "
import sys; sys.argv=['spmv_time.py','--config','c5','--fmt','4']
from paper_1406_2831_b200 import _lib; _lib.tuning(spmv_variant=$v)
import runpy; runpy.run_path('tools/spmv_time.py', run_name='__main__')" >> gpurun_out/r2s_spmv.log 2>&1; echo "variant $v" >> gpurun_out/r2s_spmv.log; done
cat gpurun_out/r2s_spmv.log
for v in 0 1 0 1; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune spmv_variant=$v >> gpurun_out/r2s_iter.log 2>&1; done
cat gpurun_out/r2s_iter.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "offset or formats" > gpurun_out/r2s_pytest.log 2>&1; tail -2 gpurun_out/r2s_pytest.log
