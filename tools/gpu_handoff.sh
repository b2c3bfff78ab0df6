timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs10.txt 2>&1; }
  LABEL=handoff_resume; run X=1
  LABEL=handoff_restart; run SCUBA_OOB_HANDOFF_RESUME=0
done; done
grep -v "^\[" gpurun_out/knobs10.txt
