SCUBA_OOB_TRACE=2 SCUBA_OOB_JIT_MIN=100000000 timeout 600 python tools/stats_run.py c3 c4 > gpurun_out/stats.log 2>&1
