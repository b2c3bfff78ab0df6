export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_api.py tests/test_gpu_multidev.py tests/test_gpu_analyzer.py -x -q 2>&1 | tail -2
timeout 600 python tools/fast_bench.py c3:100000 c4:100000 c5s:100000 c5:2000 2>&1 | grep "fast .*M q/s\|equal"
