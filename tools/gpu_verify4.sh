timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python tools/mem_probe.py 2>&1 | grep -v "^\[oob"
for c in c3 c4 c5s; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
bash tools/gpu_multirank.sh
