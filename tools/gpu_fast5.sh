export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -2
timeout 600 python tools/fast_bench.py c3:100000 c4:100000 c5s:100000 c5:2000 2>&1 | grep "M q/s\|equal"
