for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs12.txt 2>&1; }
  LABEL=base; run X=1
  LABEL=hp128; run SCUBA_OOB_HEAVY_PASSES=128
  LABEL=hp256; run SCUBA_OOB_HEAVY_PASSES=256
  LABEL=mult2; run SCUBA_OOB_JIT_GRID_MULT=2
  LABEL=mult4; run SCUBA_OOB_JIT_GRID_MULT=4
done; done
