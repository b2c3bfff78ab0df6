for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs6.txt 2>&1; }
  LABEL=base; run X=1
  LABEL=heavy_passes128; run SCUBA_OOB_HEAVY_PASSES=128
  LABEL=heavy_passes192; run SCUBA_OOB_HEAVY_PASSES=192
  LABEL=jit_min512; run SCUBA_OOB_JIT_MIN=512
  LABEL=hp128_jm512; run SCUBA_OOB_HEAVY_PASSES=128 SCUBA_OOB_JIT_MIN=512
done; done
cat gpurun_out/knobs6.txt | grep -v "^\["
