# device exhaustive oracle: parity tests, throughput, ncu of the sweep kernel
set -x
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/pytest_sweep.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_sweep.log
timeout 600 python tools/sweep_bench.py 64 256 1024 > gpurun_out/sweep_bench.jsonl 2>&1; echo "bench rc=$?"
tail -4 gpurun_out/sweep_bench.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oob_sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_full python -c "
import sys; sys.path.insert(0,'.')
from paper_2601_21552_b200 import sweep as S
p=S.load_programs('tests/golden/sweep_programs.json')['corpus/figs/push_node.mcu']
S.sweep_once(p,256,3); S.sweep_once(p,256,3)" > gpurun_out/ncu_sweep.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_sweep.log
