SCUBA_OOB_TRACE=1 timeout 600 python tools/dbg_plan.py > gpurun_out/dbg.log 2>&1
