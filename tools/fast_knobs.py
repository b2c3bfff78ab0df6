"""Fast-mode hand-off thresholds: plan-run ms for several heavy_nodes values
(SCUBA_OOB_HEAVY_PASSES from the environment).  usage: fast_knobs.py cfg n"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
fb = synth.generate(cfg, n, names=False)
base = None
for hn in [int(x) for x in os.environ.get("HN", "0,48,96,192,-1").split(",")]:
    p = _lib.Plan(fb, 30.0, flags=_lib.F_FAST, heavy_nodes=hn)
    ms = sorted(p.run() for _ in range(7))
    r = p.results()
    p.close()
    h = hash(r["verdict"].tobytes() + r["model"].tobytes())
    base = base or h
    print(f"{cfg} passes={os.environ.get('SCUBA_OOB_HEAVY_PASSES', '128')} heavy_nodes={hn}: "
          f"median {ms[3]:.2f} ms (min {ms[0]:.2f}) same={h == base}", flush=True)
