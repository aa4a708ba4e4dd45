cd $GRAFT_REPO_ROOT
for cfg in "spmv_prefetch_mb=0" "spmv_prefetch_mb=4" "spmv_prefetch_mb=8" "spmv_prefetch_mb=16" "spmv_prefetch_mb=32" "spmv_prefetch_mb=8 spmv_variant=1" "spmv_prefetch_mb=0 spmv_variant=1"; do
timeout 300 python -c "
import sys; sys.argv=['spmv_time.py','--config','c5','--fmt','4']
from paper_1406_2831_b200 import _lib; _lib.tuning(**{kv.split('=')[0]: int(kv.split('=')[1]) for kv in '$cfg'.split()})
import runpy; runpy.run_path('tools/spmv_time.py', run_name='__main__')" > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2u_spmv.log; done
cat gpurun_out/r2u_spmv.log
for cfg in "spmv_prefetch_mb=0" "spmv_prefetch_mb=8" "spmv_prefetch_mb=16" "spmv_prefetch_mb=0" "spmv_prefetch_mb=8" "spmv_prefetch_mb=16"; do timeout 900 python tools/iter_time.py --config c5 --max-itn 60 --tune $cfg > /tmp/o.txt 2>&1; echo "$cfg $(cat /tmp/o.txt)" >> gpurun_out/r2u_iter.log; done
cat gpurun_out/r2u_iter.log
