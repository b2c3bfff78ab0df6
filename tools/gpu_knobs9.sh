timeout 900 python -m pytest tests/test_gpu_jit.py -x -q 2>&1 | tail -1
for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs9.txt 2>&1; }
  LABEL=order_work; run X=1
  LABEL=order_id; run SCUBA_OOB_JIT_ORDER=0
done; done
grep -v "^\[" gpurun_out/knobs9.txt
