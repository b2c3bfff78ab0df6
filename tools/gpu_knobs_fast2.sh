export CUDA_DEVICE_MAX_CONNECTIONS=32
for hp in 32 64 128; do SCUBA_OOB_FAST_HEAVY_PASSES=$hp timeout 600 python tools/fast_knobs.py c4 100000; done
for hp in 32 64; do SCUBA_OOB_FAST_HEAVY_PASSES=$hp timeout 600 python tools/fast_knobs.py c3 100000; done
timeout 900 python -m pytest tests/test_gpu_fast.py -k frontier_prover -x -q 2>&1 | tail -2
