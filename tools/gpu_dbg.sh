rm -f gpurun_out/tl_c3.bin gpurun_out/tl_c4.bin
SCUBA_OOB_TIMELINE=gpurun_out/tl_c3.bin timeout 300 python tools/tl_run.py c3 > gpurun_out/tl.log 2>&1
python tools/timeline.py gpurun_out/tl_c3.bin 1 > gpurun_out/tl_c3.txt
SCUBA_OOB_TIMELINE=gpurun_out/tl_c4.bin timeout 300 python tools/tl_run.py c4 >> gpurun_out/tl.log 2>&1
python tools/timeline.py gpurun_out/tl_c4.bin 4 > gpurun_out/tl_c4.txt
