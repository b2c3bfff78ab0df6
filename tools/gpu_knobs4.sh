for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs4.txt 2>&1; }
  LABEL=base; run X=1
  for m in 6 12 24 48; do LABEL=mult64_$m; run SCUBA_OOB_JIT_GRID_MULT64=$m; done
done
cat gpurun_out/knobs4.txt | grep -v "^\["
