timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
SCUBA_OOB_TRACE=1 timeout 300 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
fb=synth.generate('c3',100000,names=False)
for i in range(4):
    t=time.perf_counter(); solve_flat(fb,30.0); print('solve_flat', round(1e3*(time.perf_counter()-t),1),'ms',flush=True)
" > gpurun_out/trace_c3.log 2>&1; tail -16 gpurun_out/trace_c3.log
timeout 900 python bench.py --config c3 > gpurun_out/bench_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/bench_c3.log | cut -c1-300
