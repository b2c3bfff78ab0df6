export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 300 python tools/e2e_phases.py c3 100000 fast 2>&1 | tail -18
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 2 --warmup 1 --no-extras > gpurun_out/bench_2rank.log 2>&1; echo "2-rank rc=$?"; grep -v "^\[oob\]" gpurun_out/bench_2rank.log | tail -c 1500
