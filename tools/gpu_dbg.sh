timeout 300 python tools/tl_solve.py c4 2 > /dev/null 2>&1
rm -f /tmp/tl_m.bin
SCUBA_OOB_TIMELINE=/tmp/tl_m.bin timeout 300 python tools/tl_solve.py c4 5 > gpurun_out/tl.log 2>&1
python tools/tl_w0.py /tmp/tl_m.bin 5 >> gpurun_out/tl.log
