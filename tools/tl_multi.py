"""Per-run job summary from a SCUBA_OOB_TIMELINE dump of several solve_flat calls."""
import sys
import numpy as np
r = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 10)
n = int(sys.argv[2])
# each call appends all jobs' entries; split by query-id restarts per call: use counts
per = len(r) // n
for k in range(n):
    x = r[k * per:(k + 1) * per]
    x = x[x[:, 3] != -1]
    q, wide, shadow, verdict, nodes, passes, t0, th, tf, te = x.T
    base = t0[t0 > 0].min()
    line = []
    for w in (3, 0, 1, 2):
        m = wide == w
        if m.any():
            line.append(f"w{w}: n={m.sum()} end={(te[m].max() - base) / 1e6:.1f} heavy={(th[m] > 0).sum()}")
    print(f"run {k}: span {(te.max() - base) / 1e6:.1f} ms | " + " | ".join(line))
