export CUDA_DEVICE_MAX_CONNECTIONS=32
for gm in 6 12; do echo "GRID_MULT=$gm"; SCUBA_OOB_JIT_GRID_MULT=$gm timeout 600 python tools/fast_knobs.py c3 100000 | grep "nodes=96\|nodes=-1"; SCUBA_OOB_JIT_GRID_MULT=$gm timeout 600 python tools/fast_knobs.py c4 100000 | grep "nodes=96\|nodes=-1"; done
echo "FAST_HEAVY_PASSES=512"; SCUBA_OOB_FAST_HEAVY_PASSES=512 timeout 600 python tools/fast_knobs.py c3 100000 | grep "nodes=96\|nodes=192"
