set -x
timeout 1200 python -m pytest tests/test_gpu_jit.py -x -q > gpurun_out/pytest_jit.log 2>&1; echo "pytest jit rc=$?"; tail -30 gpurun_out/pytest_jit.log
SCUBA_OOB_TRACE=1 timeout 600 python tools/trace_run.py c3 100000 > gpurun_out/trace_c3.log 2>&1; echo rc=$?
