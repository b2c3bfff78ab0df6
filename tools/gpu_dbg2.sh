export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 compute-sanitizer --tool memcheck --print-limit 2 python tools/dbg_fast.py fast 2000 2>&1 | grep -v "Host Frame" | head -40
