nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cold tools/cold_probe.cu
/tmp/cold; CUDA_DEVICE_MAX_CONNECTIONS=32 /tmp/cold; CUDA_DEVICE_MAX_CONNECTIONS=32 /tmp/cold
SCUBA_OOB_TRACE=1 CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python tools/cold_start.py fast 2>&1 | head -12
