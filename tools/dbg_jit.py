import os, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from conftest import load_golden
from paper_2601_21552_b200 import _lib
from paper_2601_21552_b200.solver import solve_flat
from paper_2601_21552_b200.wire import flatten
recs = [r for r in load_golden("synth_c3") if r["verdict"] != "timeout"]
fb = flatten(recs)
for heavy, jm, fl in ((0, 1, 0), (-1, 1, 0), (-1, 1, 0), (-1, 1, 0), (0, 1, 0), (-1, 0, _lib.F_NO_JIT)):
    print("=== heavy", heavy, "jit_min", jm, flush=True)
    out = solve_flat(fb, 30.0, heavy_nodes=heavy, jit_min=jm, flags=fl)
    bad = np.nonzero(out["verdict"] == -1)[0]
    print("status", out["status"], out["error"][:200], "unowned", len(bad), bad[:10],
          "their nodes", [recs[i]["nodes"] for i in bad[:10]], flush=True)
