# fast-mode knob sweep after the frontier abort (results hashed: identical across settings)
for kv in "BASE=1" "SCUBA_OOB_JIT_ORDER=1" "SCUBA_OOB_JIT_STREAMS=24" "SCUBA_OOB_JIT_STREAMS=8" "SCUBA_OOB_JIT_GRID_MULT=2" "SCUBA_OOB_JIT_GRID_MULT=4" "SCUBA_OOB_FAST_HEAVY_NODES=48" "SCUBA_OOB_FAST_HEAVY_NODES=192" "SCUBA_OOB_HANDOFF_GATE=0" "SCUBA_OOB_FAST_HEAVY_PASSES=64" "SCUBA_OOB_FAST_HEAVY_PASSES=256" "BASE=2"; do
  env $kv timeout 300 python tools/fast_sweep.py c3:100000 c4:100000 2>&1 | grep ' ms ' | sed "s/^/$kv: /"
done
