for c in c3 c4 c5s; do echo "== $c"; timeout 300 python tools/jit_runs.py $c 0 2>&1 | tail -3; done
for c in c3 c4 c5s; do echo "== nojit $c"; timeout 300 python tools/jit_runs.py $c -1 2>&1 | tail -2; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
