set -x
# launch list of the bench command (cold, serialised per-launch durations)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
# full capture of the int64 solve kernel on C3 and C4 (launch order: root i256, root i128, solve i256, solve i128, solve ll)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_solve_kernel --launch-skip 2 -c 1 -o gpurun_out/c3_solve_ll python tools/profile_kernels.py c3 100000 > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_solve_kernel --launch-skip 2 -c 1 -o gpurun_out/c4_solve_ll python tools/profile_kernels.py c4 100000 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
