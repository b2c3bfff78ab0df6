export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -2
timeout 600 python tools/fast_bench.py c3:100000 c4:100000 c5s:100000 c5:2000 2>&1 | grep "fast .*M q/s"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:oob_cert_kernel python tools/profile_kernels.py c3 100000 fast 2>&1 | grep -E "oob_cert|gpu__time|inst_exec" | head -12
