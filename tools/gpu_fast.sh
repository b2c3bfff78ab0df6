# fast mode on the B200: GPU tests of the fast mode, the full GPU suite, timings
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "fast tests rc=$?"; tail -15 gpurun_out/pytest_fast.log
timeout 900 python tools/fast_bench.py ${FB_ARGS} 2>&1 | tee gpurun_out/fast_bench.log | tail -20
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
fi
