# timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c3 c4 c5s; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
# one call with 1M C4 queries on one GPU (north_star batch size), verdicts of a sample vs the oracle
timeout 900 python -c "
import sys,time; sys.path.insert(0,'.')
import numpy as np
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
from oracle import oracle
fb=synth.generate('c4',1000000,names=False)
t=time.perf_counter(); o=solve_flat(fb,30.0); dt=time.perf_counter()-t
t=time.perf_counter(); o=solve_flat(fb,30.0); dt2=time.perf_counter()-t
s=fb.slice(0,20000); r=oracle.solve_flat(s,30.0,threads=16)
print('c4 1M one call: %.2f s (warm %.2f s) -> %.0f q/s e2e; status %d; sample verdict/node mismatches %d' % (dt, dt2, 1e6/dt2, o['status'], int((r['verdict']!=o['verdict'][:20000]).sum()+(r['nodes']!=o['nodes'][:20000]).sum())))
" 2>&1 | grep -v "^\[oob" | tail -2
