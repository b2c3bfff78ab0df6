timeout 1500 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_jit128.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_jit128.log
timeout 600 python tools/critical_jit.py c4 34146 2>&1 | grep -v "^\[oob" | head -2
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" 0 >> gpurun_out/knobs8.txt 2>&1; }
  LABEL=jit128; run X=1
  LABEL=no_jit128; run SCUBA_OOB_JIT128=0
  LABEL=jit128_b; run X=1
done
grep -v "^\[" gpurun_out/knobs8.txt
