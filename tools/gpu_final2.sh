timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 python bench.py --config c5s > gpurun_out/bench_c5s.log 2>&1; echo "c5s rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
bash tools/gpu_multirank.sh
