# opt-in warp-per-query search (OOB_F_CHAIN, chain.cuh): GPU tests, A/B against
# the default fast mode, one --set full capture of the search kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/chain_pytest.log 2>&1; echo "pytest fast rc=$?"; tail -3 gpurun_out/chain_pytest.log
SCUBA_OOB_CHAIN=1 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 2>&1 | tail -8
SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 2>&1 | tail -4
SCUBA_OOB_CHAIN=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:oob_chain_kernel -c 1 -o gpurun_out/r02_chain_full python tools/profile_kernels.py c3 100000 fast > gpurun_out/ncu_chain.log 2>&1; echo "ncu chain rc=$?"
