# host-phase trace of the e2e call + bench lines for C4 / C5s with the current bench
set -x
SCUBA_OOB_TRACE=1 timeout 300 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
fb=synth.generate('c3',100000,names=False)
for i in range(4):
    t=time.perf_counter(); solve_flat(fb,30.0); print('solve_flat', round(1e3*(time.perf_counter()-t),1),'ms',flush=True)
" > gpurun_out/trace_c3.log 2>&1
tail -40 gpurun_out/trace_c3.log
timeout 600 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/bench_c3.log
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/bench_c4.log
timeout 600 python bench.py --config c5s > gpurun_out/bench_c5s.log 2>&1; echo "c5s rc=$?"; tail -1 gpurun_out/bench_c5s.log
