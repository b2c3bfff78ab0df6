for rep in 1 2 3; do
for cfg in c3 c4; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs15.txt 2>&1; }
  LABEL=streams16; run X=1
  LABEL=streams20; run SCUBA_OOB_JIT_STREAMS=20
  LABEL=streams24; run SCUBA_OOB_JIT_STREAMS=24
done; done
