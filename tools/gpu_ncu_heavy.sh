# --set full of the longest compiled-class launch of a C3 fast plan run (the
# heavy Sat chains; launch index from profiles/r02_launches_c3_fast.csv)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_jit_solve --launch-skip ${SKIP:-56} -c 1 -o gpurun_out/r02_jit_heavy_full python tools/profile_kernels.py c3 100000 fast > gpurun_out/ncu_heavy.log 2>&1; echo "ncu heavy rc=$?"; tail -3 gpurun_out/ncu_heavy.log
