# knob sweep of the solve engine (plan-run device time, C3 and C4)
for cfg in c3 c4; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" $HN >> gpurun_out/knobs.txt 2>&1; }
  HN=0
  LABEL=base; run X=1
  LABEL=base2; run X=1
  LABEL=heavy_passes128; run SCUBA_OOB_HEAVY_PASSES=128
  LABEL=heavy_passes512; run SCUBA_OOB_HEAVY_PASSES=512
  LABEL=heavy_passes1024; run SCUBA_OOB_HEAVY_PASSES=1024
  LABEL=grid_mult2; run SCUBA_OOB_JIT_GRID_MULT=2
  LABEL=jit_warps4; run SCUBA_OOB_JIT_WARPS=4
  LABEL=maxreg96; run SCUBA_OOB_JIT_MAXREG=96
  LABEL=maxreg128; run SCUBA_OOB_JIT_MAXREG=128
  LABEL=wait5ms; run SCUBA_OOB_FRONTIER_WAIT_US=5000
  LABEL=wait50ms; run SCUBA_OOB_FRONTIER_WAIT_US=50000
  LABEL=streams8; run SCUBA_OOB_JIT_STREAMS=8
  LABEL=streams32; run SCUBA_OOB_JIT_STREAMS=32
  LABEL=x32_first; run SCUBA_OOB_X32_FIRST=1
  LABEL=jit_min512; run SCUBA_OOB_JIT_MIN=512
  LABEL=jit_min4096; run SCUBA_OOB_JIT_MIN=4096
  HN=8; LABEL=heavy_nodes8; run X=1
  HN=32; LABEL=heavy_nodes32; run X=1
  HN=64; LABEL=heavy_nodes64; run X=1
done
cat gpurun_out/knobs.txt
