rm -f gpurun_out/tl_c4.bin
SCUBA_OOB_TIMELINE=gpurun_out/tl_c4.bin timeout 300 python tools/tl_run.py c4 > gpurun_out/tl.log 2>&1
python tools/timeline.py gpurun_out/tl_c4.bin 10 > gpurun_out/tl_c4.txt
