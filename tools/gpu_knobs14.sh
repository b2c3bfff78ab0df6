for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs14.txt 2>&1; }
  LABEL=base; run X=1
  LABEL=jm512; run SCUBA_OOB_JIT_MIN=512
  LABEL=jm2048; run SCUBA_OOB_JIT_MIN=2048
  LABEL=streams24; run SCUBA_OOB_JIT_STREAMS=24
  LABEL=streams12; run SCUBA_OOB_JIT_STREAMS=12
done; done
