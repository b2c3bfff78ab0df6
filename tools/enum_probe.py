import sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from conftest import load_golden, VCODE
from paper_2601_21552_b200 import _lib
from paper_2601_21552_b200.solver import solve_flat
from paper_2601_21552_b200.wire import flatten
for name in ["random_solver", "random_accept", "crafted"]:
    recs = [r for r in load_golden(name) if r["verdict"] != "timeout" and r["timeout"] >= 1.0]
    fb = flatten(recs)
    out = solve_flat(fb, 30.0, flags=_lib.F_FAST)
    gn = np.array([r["nodes"] for r in recs])
    print(os.environ.get("SCUBA_OOB_ENUM_MAX"), name, "nodes==0 & gold>0:", int(((out["nodes"] == 0) & (gn > 0)).sum()),
          "unsat", int((out["verdict"] == 0).sum()))
    rg = _lib.query_regimes(fb) if hasattr(_lib, "query_regimes") else None
    if rg is not None: print("  regimes", np.bincount(rg.astype(np.int64)))
