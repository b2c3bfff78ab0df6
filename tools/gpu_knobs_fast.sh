export CUDA_DEVICE_MAX_CONNECTIONS=32
for hp in 128 512 4096; do SCUBA_OOB_HEAVY_PASSES=$hp timeout 600 python tools/fast_knobs.py c3 100000; done
for hp in 128 512; do SCUBA_OOB_HEAVY_PASSES=$hp timeout 600 python tools/fast_knobs.py c4 100000; done
