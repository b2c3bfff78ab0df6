# ncu evidence for the round-2 workloads: launch lists with DRAM bytes and warp
# instructions per kernel (one plan run each), then --set full captures of the
# certificate kernel and of the first compiled-class kernel in fast mode
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=16
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for spec in "c3 100000 fast" "c3 100000 canonical" "c4 100000 fast" "c5 2000 fast" "c5s 100000 fast"; do
  set -- $spec
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/traffic_$1_$3_$2.csv python tools/profile_kernels.py $1 $2 $3 > /dev/null 2>&1; echo "ncu $spec rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_cert_kernel -c 1 -o gpurun_out/r02_cert_full python tools/profile_kernels.py c3 100000 fast > gpurun_out/ncu_full1.log 2>&1; echo "full cert rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_solve_kernel -c 1 -o gpurun_out/r02_solve_fast_full python tools/profile_kernels.py c3 100000 fast > gpurun_out/ncu_full3.log 2>&1; echo "full solve rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/b_ncu.log 2>&1; echo "bench launch list rc=$?"
