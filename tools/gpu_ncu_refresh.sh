timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_quick.log 2>&1; echo "bench quick rc=$?"; tail -c 600 gpurun_out/bench_quick.log
bash tools/gpu_ncu_r02.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_jit_solve -c 1 -o gpurun_out/r02_jit_fast_full python tools/profile_kernels.py c3 100000 fast > gpurun_out/ncu_full4.log 2>&1; echo "full jit rc=$?"
ls gpurun_out
