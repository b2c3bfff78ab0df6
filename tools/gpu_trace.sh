set -x
SCUBA_OOB_TRACE=1 timeout 600 python tools/trace_run.py c3 100000 > gpurun_out/trace_c3.log 2>&1; echo rc=$?
SCUBA_OOB_TRACE=1 timeout 600 python tools/trace_run.py c4 100000 > gpurun_out/trace_c4.log 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_kernels.py c3 100000 > /dev/null 2>&1; echo rc=$?
