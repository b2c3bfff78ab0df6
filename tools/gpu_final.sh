timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in c3 c4 c5s; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "list rc=$?"
for cfg in c3 c4; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/traffic_$cfg.csv python tools/profile_kernels.py $cfg 100000 > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done
