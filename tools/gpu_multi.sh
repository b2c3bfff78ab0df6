export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_multidev.py -x -q 2>&1 | tail -3
timeout 300 python tools/e2e_phases.py c3 100000 fast 2>&1 | tail -32
