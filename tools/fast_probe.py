"""Where the fast mode's time goes on a synthetic config: the Sat-only
sub-batch under the canonical engine, and the certificate kernel alone
(every query of a Sat-free stream).  usage: python tools/fast_probe.py [cfg n]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402
from paper_2601_21552_b200.wire import flatten  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
fb = synth.generate(cfg, n, names=True)
p = _lib.Plan(fb, 30.0, flags=_lib.F_FAST)
ms = sorted(p.run() for _ in range(5))
v = p.results()["verdict"]
p.close()
print(f"{cfg} fast full: {ms[2]:.2f} ms; sat {int((v == 1).sum())}", flush=True)
sat = np.nonzero(v == 1)[0]
sub = flatten([fb.query_json(int(q)) for q in sat])
for flags, name in ((0, "canonical"), (_lib.F_FAST, "fast")):
    p = _lib.Plan(sub, 30.0, flags=flags)
    ms = sorted(p.run() for _ in range(5))
    p.close()
    print(f"{cfg} Sat-only sub-batch ({sub.n}) {name}: {ms[2]:.2f} ms", flush=True)
