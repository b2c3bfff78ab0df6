nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/alu_peak tools/alu_peak.cu && /tmp/alu_peak > gpurun_out/alu_peak.jsonl; cat gpurun_out/alu_peak.jsonl
for cfg in c3 c4; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/traffic_$cfg.csv python tools/profile_kernels.py $cfg 100000 > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_jit_solve --launch-skip 11 -c 1 -o gpurun_out/jit_top_c3 python tools/profile_kernels.py c3 100000 > gpurun_out/ncu_jit.log 2>&1; echo "full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "list rc=$?"
