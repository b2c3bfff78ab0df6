for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" $HN >> gpurun_out/knobs13.txt 2>&1; }
  HN=0; LABEL=base; run X=1
  HN=0; LABEL=hp96; run SCUBA_OOB_HEAVY_PASSES=96
  HN=20; LABEL=hn20; run X=1
  HN=28; LABEL=hn28; run X=1
  HN=0; LABEL=wait5ms; run SCUBA_OOB_FRONTIER_WAIT_US=5000
done; done
