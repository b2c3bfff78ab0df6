# frontier: per-round pass cap of the speculative lanes (SCUBA_OOB_FRONTIER_SPEC_CAP), fast mode + parity with it on
mkdir -p gpurun_out
SCUBA_OOB_FRONTIER_SPEC_CAP=16 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fast.py -x -q > gpurun_out/fs_pytest.log 2>&1; echo "pytest (cap 16) rc=$?"; tail -2 gpurun_out/fs_pytest.log
for c in 0 8 16 32 64 0; do
  SCUBA_OOB_FRONTIER_SPEC_CAP=$c timeout 300 python tools/fast_sweep.py c3:100000 c4:100000 c5s:100000 2>&1 | grep ' ms ' | sed "s/^/cap=$c: /"
done
