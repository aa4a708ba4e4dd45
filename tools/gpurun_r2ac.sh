cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 1; do timeout 600 python tools/spmm_time.py --config c5 --ncols 30 --tune spmm_variant=$v >> gpurun_out/r2ac_spmm.log 2>&1; done
cat gpurun_out/r2ac_spmm.log
for v in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "offset or shared or formats" --co -q > /dev/null 2>&1; KRB_X=1 timeout 600 python -c "
from paper_1406_2831_b200 import _lib; _lib.tuning(spmm_variant=$v)
import pytest, sys; sys.exit(pytest.main(['-q','-x','tests/test_gpu_kernels.py','-k','offset or shared or formats']))" > /tmp/o.txt 2>&1; echo "variant $v $(tail -1 /tmp/o.txt)" >> gpurun_out/r2ac_pytest.log; done
cat gpurun_out/r2ac_pytest.log
