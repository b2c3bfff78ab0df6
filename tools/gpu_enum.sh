# fast-mode K3 enumeration (chain.cuh oob_enum_kernel): GPU tests, A/B timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/enum_pytest.log 2>&1; echo "pytest fast rc=$?"; tail -15 gpurun_out/enum_pytest.log
SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 c5s:100000 2>&1 | grep chain= | cut -c1-150
SCUBA_OOB_ENUM_MAX=0 SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 c5s:100000 2>&1 | grep chain= | cut -c1-150 | sed 's/^/enum off /'
