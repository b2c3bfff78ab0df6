timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs7.txt 2>&1; }
  LABEL=hp192_perwarp; run X=1
  LABEL=hp256_perwarp; run SCUBA_OOB_HEAVY_PASSES=256
  LABEL=hp128_perwarp; run SCUBA_OOB_HEAVY_PASSES=128
  LABEL=hp192_slabpool; run SCUBA_OOB_SLAB_POOL=1
  LABEL=hp256_slabpool; run SCUBA_OOB_SLAB_POOL=1 SCUBA_OOB_HEAVY_PASSES=256
done; done
cat gpurun_out/knobs7.txt | grep -v "^\["
