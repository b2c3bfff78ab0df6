# The reference's own test suite (baseline/_ref/tests, copied by
# tools/install_reference.sh) with every solve() decided by the CUDA engine
# (tools/ref_patch_gpu.py), in both modes.  Run on the GPU box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for mode in canonical fast; do
  SCUBA_REF_SUITE_MODE=$mode PYTHONPATH="$PWD/tools:$PWD/baseline/_ref" timeout 1800 python -m pytest -p ref_patch_gpu \
    baseline/_ref/tests -q -p no:cacheprovider > gpurun_out/ref_suite_gpu_$mode.log 2>&1
  echo "reference suite on the GPU engine ($mode) rc=$?"; tail -3 gpurun_out/ref_suite_gpu_$mode.log; grep "solve() calls" gpurun_out/ref_suite_gpu_$mode.log
done
