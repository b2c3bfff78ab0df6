export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python tools/fast_probe.py c3 100000 2>&1 | tail -5
SCUBA_OOB_TRACE=1 timeout 600 python tools/fast_bench.py c3:100000 2>&1 | grep -v "pack\|pool" | head -40
