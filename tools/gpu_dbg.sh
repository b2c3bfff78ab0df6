for ch in 0 16384 25000 34000 50000; do SCUBA_OOB_CHUNK=$ch timeout 300 python tools/e2e_sweep.py c3; done > gpurun_out/e2e.log 2>&1
for ch in 0 34000; do SCUBA_OOB_CHUNK=$ch timeout 300 python tools/e2e_sweep.py c4; done >> gpurun_out/e2e.log 2>&1
