# frontier: speculative-lane abort (SCUBA_OOB_FRONTIER_ABORT) -- parity suites with it on, then A/B
mkdir -p gpurun_out
SCUBA_OOB_FRONTIER_ABORT=2 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fast.py tests/test_gpu_jit.py -x -q > gpurun_out/fa_pytest.log 2>&1; echo "pytest (abort 2) rc=$?"; tail -3 gpurun_out/fa_pytest.log
for f in 0 2 4 8; do
  SCUBA_OOB_FRONTIER_ABORT=$f SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 c5s:100000 2>&1 | grep chain= | cut -c1-175 | sed "s/^/fa=$f /"
done
