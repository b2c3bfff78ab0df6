SCUBA_OOB_TRACE=1 timeout 600 python tools/e2e_sweep.py c3 > gpurun_out/trace_pk.log 2>&1
