import sys
import numpy as np
r = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 10)
n = int(sys.argv[2]); per = len(r) // n
for k in range(n):
    x = r[k * per:(k + 1) * per]
    x = x[x[:, 3] != -1]
    q, wide, shadow, verdict, nodes, passes, t0, th, tf, te = x.T
    base = t0[t0 > 0].min()
    m = np.nonzero(wide == 0)[0]
    o = m[np.argsort(-(te[m]))[:6]]
    print(f"run {k} span {(te.max()-base)/1e6:.1f}")
    for i in o:
        f = lambda t: (t - base) / 1e6 if t > 0 else -1
        print(f"   q={q[i]} sh={shadow[i]} nodes={nodes[i]} passes={passes[i]} start={f(t0[i]):.1f} handoff={f(th[i]):.1f} fstart={f(tf[i]):.1f} end={f(te[i]):.1f}")
