import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_21552_b200 import _lib, synth
from paper_2601_21552_b200.solver import solve_flat
fb = synth.generate("c3", 5000, names=False)
ref = solve_flat(fb, 30.0, flags=_lib.F_NO_JIT)
s64 = solve_flat(fb, 30.0, jit_min=64)
print("solve jit64 vs ref verdict mism", int((s64["verdict"] != ref["verdict"]).sum()), flush=True)
for runs in (1, 2, 3):
    p = _lib.Plan(fb, 30.0, jit_min=64)
    for _ in range(runs):
        p.run()
    r = p.results()
    bad = np.nonzero(r["verdict"] != ref["verdict"])[0]
    print("runs", runs, "mism", len(bad), bad[:8], r["verdict"][bad[:8]], ref["verdict"][bad[:8]],
          "nodes mism", int((r["nodes"] != ref["nodes"]).sum()), flush=True)
    del p
for runs in (1, 2):
    p = _lib.Plan(fb, 30.0, flags=_lib.F_NO_JIT)
    for _ in range(runs):
        p.run()
    r = p.results()
    print("nojit plan runs", runs, "mism", int((r["verdict"] != ref["verdict"]).sum()), flush=True)
