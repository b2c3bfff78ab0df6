"""Fast-mode plan-run time of C3/C4 under the current environment's knobs,
with a hash of the results (verdicts, models) to check they are identical.
usage: KNOBS... python tools/fast_sweep.py [cfg:n ...]"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

out = []
for spec in sys.argv[1:] or ["c3:100000", "c4:100000"]:
    cfg, n = spec.split(":")
    fb = synth.generate(cfg, int(n), names=False)
    p = _lib.Plan(fb, 30.0, flags=_lib.F_FAST)
    ms = sorted(p.run() for _ in range(9))
    r = p.results()
    p.close()
    h = hashlib.sha1(r["verdict"].tobytes() + r["model"].tobytes()).hexdigest()[:10]
    out.append(f"{cfg} {np.median(ms):.3f} ms [{ms[1]:.3f}-{ms[-2]:.3f}] {h}")
print(" | ".join(out), flush=True)
