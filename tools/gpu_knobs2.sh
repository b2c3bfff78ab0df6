for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs2.txt 2>&1; }
  LABEL=base; run X=1
  for m in 2 3 4 6 8; do LABEL=grid_mult$m; run SCUBA_OOB_JIT_GRID_MULT=$m; done
  LABEL=grid_mult3_streams32; run SCUBA_OOB_JIT_GRID_MULT=3 SCUBA_OOB_JIT_STREAMS=32
  LABEL=grid_mult3_maxreg96; run SCUBA_OOB_JIT_GRID_MULT=3 SCUBA_OOB_JIT_MAXREG=96
done
cat gpurun_out/knobs2.txt | grep -v "^\["
