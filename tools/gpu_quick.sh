# quick GPU iteration: parity suite + smoke + host trace + one bench line
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
SCUBA_OOB_TRACE=1 timeout 600 python tools/trace_run.py c3 100000 2>&1 | head -60 > gpurun_out/trace_c3.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
timeout 300 python tools/jit_runs.py c4 0 > gpurun_out/c4runs.log 2>&1; tail -2 gpurun_out/c4runs.log
