"""Where a fast-mode step's time goes: one plan run with per-entry device
timestamps (SCUBA_OOB_TIMELINE) -> step time, the search span, and the
longest entries (query, job, nodes, passes, duration).
usage: python tools/tl_tail.py [cfg] [n]"""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
path = os.path.join(tempfile.mkdtemp(), "tl.bin")
os.environ["SCUBA_OOB_TIMELINE"] = path
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
fb = synth.generate(cfg, n, names=False)
plan = _lib.Plan(fb, 30.0, n_gpus=1, device=0, flags=_lib.F_FAST)
for _ in range(2):
    plan.run()
open(path, "wb").close()
ms = plan.run()
plan.results()
r = np.fromfile(path, dtype=np.int64).reshape(-1, 10)
r = r[r[:, 3] != -1]
q, wide, shadow, verdict, nodes, passes, t0, th, tf, te = r.T
m = t0 > 0
base = t0[m].min()
print(f"step {ms:.3f} ms; searched entries {int(m.sum())}; search span {(te[m].max() - base) / 1e6:.3f} ms")
d = (te - t0) / 1e6
for i in np.argsort(-d * m)[:12]:
    print(f"  q {q[i]:6d} job {wide[i]} shadow {shadow[i]} verdict {verdict[i]} nodes {nodes[i]:5d} passes {passes[i]:6d} "
          f"start {(t0[i] - base) / 1e6:.3f} dur {d[i]:.3f} ms heavy {th[i] > 0}")
