set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/tl_c3.bin gpurun_out/tl_c4.bin
SCUBA_OOB_TIMELINE=gpurun_out/tl_c3.bin timeout 300 python tools/profile_kernels.py c3 100000 > gpurun_out/tl.log 2>&1
SCUBA_OOB_TIMELINE=gpurun_out/tl_c4.bin timeout 300 python tools/profile_kernels.py c4 100000 >> gpurun_out/tl.log 2>&1
python tools/timeline.py gpurun_out/tl_c3.bin > gpurun_out/tl_c3.txt
python tools/timeline.py gpurun_out/tl_c4.bin 20 > gpurun_out/tl_c4.txt
