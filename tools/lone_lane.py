"""Lone-lane pass latency: one long-chain query alone on the GPU, interpreted
and compiled (run on the GPU box)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_21552_b200 import _lib, synth
fb = synth.generate("c3", 100000, names=False)
q = int(sys.argv[1]) if len(sys.argv) > 1 else 91976
one = fb.slice(q, q + 1)
for name, kw in (("interp", dict(flags=_lib.F_NO_JIT, heavy_nodes=-1)), ("jit", dict(jit_min=1, heavy_nodes=-1))):
    p = _lib.Plan(one, 30.0, **kw)
    ms = [p.run() for _ in range(5)]
    r = p.results()
    print(name, "passes", int(r["passes"][0]), "nodes", int(r["nodes"][0]), "ms", [round(x, 3) for x in ms],
          "us/pass %.2f" % (1e3 * min(ms) / max(1, int(r["passes"][0]))), flush=True)
