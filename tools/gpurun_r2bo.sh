cd $GRAFT_REPO_ROOT
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "value_coded or offset_coded_format_choice or value_coding" > gpurun_out/r2bo_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -6 gpurun_out/r2bo_memcheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -k "value_coding" > gpurun_out/r2bo_memcheck2.log 2>&1; echo "memcheck2 rc=$?"; tail -4 gpurun_out/r2bo_memcheck2.log
