mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "fast tests rc=$?"; tail -15 gpurun_out/pytest_fast.log
SCUBA_OOB_TRACE=2 timeout 600 python tools/fast_bench.py c3:100000 c4:100000 c5s:100000 c5:2000 > gpurun_out/fb.log 2>&1; echo rc=$?
grep "fast mode\|M q/s\|rror\|certify\|equal" gpurun_out/fb.log | grep -v "w1: \|w2: \|w3: " | tail -40
