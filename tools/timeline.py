"""Summarise a SCUBA_OOB_TIMELINE dump (one solve run).

    python tools/timeline.py <file> [bucket_ms]
"""
import sys

import numpy as np

path = sys.argv[1]
bucket = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
r = np.fromfile(path, dtype=np.int64).reshape(-1, 10)
r = r[r[:, 3] != -1]  # owned entries only
q, wide, shadow, verdict, nodes, passes, t0, th, tf, te = r.T
base = t0[t0 > 0].min()
ms = lambda t: (t - base) / 1e6
end = ms(te.max())
print(f"entries {len(r)}  span {end:.2f} ms  heavy {int((th > 0).sum())}")
heavy = th > 0
ls_end = np.where(heavy, th, te)
print(f"last lockstep finish {ms(ls_end.max()):.2f} ms; frontier: first claim {ms(tf[heavy].min()) if heavy.any() else 0:.2f} "
      f"last end {ms(te[heavy].max()) if heavy.any() else 0:.2f}")
nb = int(end / bucket) + 1
lock = np.zeros(nb)
front = np.zeros(nb)
wait = np.zeros(nb)
for a, b, arr in ((t0, ls_end, lock), (th, tf, wait), (tf, te, front)):
    m = (a > 0) & (b > 0)
    for x, y in zip(ms(a[m]), ms(b[m])):
        i0, i1 = int(x / bucket), int(y / bucket)
        arr[i0:i1 + 1] += 1
print(" t(ms)  lockstep-lanes  queued  frontier-queries")
for i in range(nb):
    print(f"{i * bucket:6.1f}  {lock[i]:8.0f}  {wait[i]:6.0f}  {front[i]:6.0f}")
d = ms(te) - ms(np.where(heavy, tf, t0))
order = np.argsort(-d)[:12]
print("longest (ms from own start): q wide heavy nodes passes dur start")
for i in order:
    print(f"  {q[i]:7d} {wide[i]} {int(heavy[i])} {nodes[i]:6d} {passes[i]:6d} {d[i]:7.2f} {ms(np.where(heavy, tf, t0)[i]):7.2f}")
order = np.argsort(-te)[:12]
print("last to finish: q wide shadow heavy nodes passes end_ms frontier_start_ms")
for i in order:
    print(f"  {q[i]:7d} {wide[i]} {shadow[i]} {int(heavy[i])} {nodes[i]:6d} {passes[i]:6d} {ms(te[i]):7.2f} "
          f"{ms(tf[i]) if tf[i] > 0 else -1:7.2f}")
