export CUDA_DEVICE_MAX_CONNECTIONS=32
for g in 1 0; do echo "GATE=$g"; SCUBA_OOB_HANDOFF_GATE=$g timeout 600 python tools/fast_knobs.py c3 100000 | grep "nodes=0\|nodes=96\|nodes=-1"; SCUBA_OOB_HANDOFF_GATE=$g timeout 600 python tools/fast_knobs.py c4 100000 | grep "nodes=0\|nodes=96\|nodes=-1"; done
