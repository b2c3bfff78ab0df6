for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs5.txt 2>&1; }
  LABEL=slab_pool; run X=1
  LABEL=slab_per_warp; run SCUBA_OOB_SLAB_POOL=0
done; done
cat gpurun_out/knobs5.txt | grep -v "^\["
