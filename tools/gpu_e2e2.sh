export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_api.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_e2e.log
