timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python tools/e2e_concurrent.py c3 100000 12 > gpurun_out/e2e_conc.txt 2>&1; cat gpurun_out/e2e_conc.txt
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 300 python tools/knob_run.py $cfg 100000 "$LABEL" $HN >> gpurun_out/knobs3.txt 2>&1; }
  HN=0
  LABEL=m3_base; run X=1
  LABEL=m3_heavy_passes128; run SCUBA_OOB_HEAVY_PASSES=128
  LABEL=m3_heavy_passes512; run SCUBA_OOB_HEAVY_PASSES=512
  LABEL=m3_jit_min512; run SCUBA_OOB_JIT_MIN=512
  LABEL=m3_jit_min2048; run SCUBA_OOB_JIT_MIN=2048
  LABEL=m6_warps4; run SCUBA_OOB_JIT_GRID_MULT=6 SCUBA_OOB_JIT_WARPS=4
  LABEL=m3_wait5ms; run SCUBA_OOB_FRONTIER_WAIT_US=5000
  HN=32; LABEL=m3_heavy_nodes32; run X=1
  HN=12; LABEL=m3_heavy_nodes12; run X=1
done
cat gpurun_out/knobs3.txt | grep -v "^\["
