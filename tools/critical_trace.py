"""Frontier statistics (SCUBA_OOB_TRACE=2) of the heaviest query of a config,
decided alone: rounds, units, lane efficiency."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
q = int(sys.argv[2]) if len(sys.argv) > 2 else 94026
fb = synth.generate(cfg, 100000, names=False)
one = _lib.Plan(fb.slice(q, q + 1), 30.0)
one.run()
print("alone ms", round(min(one.run() for _ in range(2)), 2), flush=True)
r = one.results()
print("passes", int(r["passes"][0]), "nodes", int(r["nodes"][0]), "verdict", int(r["verdict"][0]), flush=True)
