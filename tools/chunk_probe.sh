for ch in 0 50000 34000 25000; do
for cfg in c3 c4; do
SCUBA_OOB_CHUNK=$ch timeout 300 python -c "
import sys,time,statistics; sys.path.insert(0,'.')
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
fb=synth.generate('$cfg',100000,names=False)
ref=solve_flat(fb,30.0)
for i in range(2): solve_flat(fb,30.0)
ts=[]
for i in range(6):
    t=time.perf_counter(); o=solve_flat(fb,30.0); ts.append(time.perf_counter()-t)
    assert (o['verdict']==ref['verdict']).all() and (o['nodes']==ref['nodes']).all()
print('$cfg chunk=$ch median %.1f ms min %.1f ms' % (1e3*statistics.median(ts), 1e3*min(ts)), flush=True)
" 2>&1 | tail -1
done; done
