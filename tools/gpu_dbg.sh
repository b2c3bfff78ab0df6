rm -f /tmp/tl_c3.bin
SCUBA_OOB_TIMELINE=/tmp/tl_c3.bin timeout 300 python tools/tl_run.py c3 > gpurun_out/tl.log 2>&1
python tools/timeline.py /tmp/tl_c3.bin 1 > gpurun_out/tl_c3.txt
SCUBA_OOB_TRACE=2 timeout 600 python tools/stats_run.py c3 > gpurun_out/stats.log 2>&1
