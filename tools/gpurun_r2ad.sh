cd $GRAFT_REPO_ROOT
for cfg in "pdl=0" "pdl=1" "pdl=0" "pdl=1"; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2ad_iter.log; done
for cfg in "pdl=0" "pdl=1"; do timeout 900 python tools/iter_time.py --config c3 c4 --system 1 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2ad_iter.log; done
cat gpurun_out/r2ad_iter.log
timeout 900 python -c "
from paper_1406_2831_b200 import _lib; _lib.tuning(pdl=1)
import pytest, sys; sys.exit(pytest.main(['-q','-x','tests/test_gpu_solvers.py','tests/test_gpu_fullsize.py','tests/test_gpu_edge.py']))" > gpurun_out/r2ad_pytest.log 2>&1; tail -2 gpurun_out/r2ad_pytest.log
timeout 600 python tools/spmm_time.py --config c5 --ncols 30 >> gpurun_out/r2ad_spmm.log 2>&1; cat gpurun_out/r2ad_spmm.log
