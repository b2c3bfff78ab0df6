# --set full of the longest compiled-class launch of a C4 fast plan run
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_jit_solve --launch-skip ${SKIP:-42} -c 1 -o gpurun_out/r02_jit_heavy_c4_full python tools/profile_kernels.py c4 100000 fast > gpurun_out/ncu_heavy_c4.log 2>&1; echo "ncu heavy c4 rc=$?"; tail -2 gpurun_out/ncu_heavy_c4.log
