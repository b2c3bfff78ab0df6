# One GPU iteration (run under gpurun): full GPU suite, smoke, both bench arms.
#   SKIP_TESTS=1 skip the test suite;  BENCH_ARGS extra bench.py flags
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -5 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
fi
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 5000 gpurun_out/bench.log
if [ -z "$SKIP_REF" ]; then
  timeout 900 python bench.py --impl reference ${BENCH_ARGS} > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"; tail -c 2000 gpurun_out/bench_ref.log
fi
