export CUDA_DEVICE_MAX_CONNECTIONS=32
for k in 4 16 64; do SCUBA_OOB_JIT_WARPS=8 SCUBA_OOB_JIT_STREAMS=$k timeout 300 python tools/jit_runs.py c3 1024 2>&1 | tail -3 | sed "s/^/c3 K=$k /"; done > gpurun_out/runs.log
for k in 4 16 64; do SCUBA_OOB_JIT_WARPS=8 SCUBA_OOB_JIT_STREAMS=$k timeout 300 python tools/jit_runs.py c4 1024 2>&1 | tail -3 | sed "s/^/c4 K=$k /"; done >> gpurun_out/runs.log
timeout 300 python tools/jit_runs.py c3 -1 2>&1 | tail -2 | sed "s/^/c3 interp /" >> gpurun_out/runs.log
