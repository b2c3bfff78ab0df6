set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
SCUBA_OOB_TRACE=1 timeout 600 python tools/trace_run.py c3 100000 2>&1 | head -30 > gpurun_out/trace_c3.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"oob_lockstep_kernel|oob_frontier_kernel" --launch-skip 4 -c 2 -o gpurun_out/c3_full python tools/profile_kernels.py c3 100000 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
