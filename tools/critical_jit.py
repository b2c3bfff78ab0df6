"""The heaviest query of a config decided alone through the interpreter and
through a compiled class (jit_min = 1), and the full step at jit_min 1."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
q = int(sys.argv[2]) if len(sys.argv) > 2 else 94026
fb = synth.generate(cfg, 100000, names=False)
for jm in (0, 1):
    one = _lib.Plan(fb.slice(q, q + 1), 30.0, jit_min=jm)
    one.run()
    ms = min(one.run() for _ in range(3))
    r = one.results()
    print(f"{cfg} q{q} jit_min={jm}: alone {ms:.2f} ms passes {int(r['passes'][0])} nodes {int(r['nodes'][0])}",
          flush=True)
    one.close()
# how many queries share the class of q (the compile threshold is per class)
import collections
sig = lambda i: (int(fb.node_begin[i + 1] - fb.node_begin[i]), int(fb.con_begin[i + 1] - fb.con_begin[i]),
                 bytes(fb.node_op[fb.node_begin[i]:fb.node_begin[i + 1]]))
s = sig(q)
print("queries with the same shape signature:", sum(1 for i in range(fb.n) if sig(i) == s), flush=True)
for jm in (0, 64):
    p = _lib.Plan(fb, 30.0, jit_min=jm)
    p.run()
    print(f"{cfg} full step jit_min={jm}: {min(p.run() for _ in range(3)):.2f} ms", flush=True)
    p.close()
