"""Critical path of a synthetic step: the queries with the most propagation
passes, each decided ALONE (one-query plans) -- a lower bound on the step time
that no scheduling can beat, since a query's passes are sequential (each pass
narrows with the previous one's domains, solver.py:271-277)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

for cfg in sys.argv[1:] or ["c3", "c4"]:
    fb = synth.generate(cfg, 100000, names=False)
    p = _lib.Plan(fb, 30.0)
    p.run()
    full = min(p.run() for _ in range(3))
    r = p.results()
    p.close()
    order = np.argsort(-r["passes"])[:5]
    for q in order:
        one = _lib.Plan(fb.slice(int(q), int(q) + 1), 30.0)
        one.run()
        ms = min(one.run() for _ in range(3))
        one.close()
        print(f"{cfg}: step {full:.2f} ms; query {q}: passes {int(r['passes'][q])} nodes {int(r['nodes'][q])} "
              f"alone {ms:.2f} ms ({1e3 * ms / max(int(r['passes'][q]), 1):.2f} us/pass)", flush=True)
