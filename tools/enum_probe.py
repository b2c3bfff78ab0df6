"""Fast-mode K3 on the golden sets: Unsat records no certificate refutes
(host build of the certificate checker) and how many of them the
enumeration decides without search.
usage: python tools/enum_probe.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))
import test_symbolic_host as H  # noqa: E402
from conftest import GOLDEN_SETS, load_golden  # noqa: E402
from paper_2601_21552_b200 import _lib  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402
from paper_2601_21552_b200.wire import flatten  # noqa: E402

H.prover.__wrapped__()
for name in GOLDEN_SETS:
    recs = [r for r in load_golden(name) if r["verdict"] != "timeout" and r["timeout"] >= 1.0]
    fb = flatten(recs)
    out = solve_flat(fb, 30.0, flags=_lib.F_FAST)
    unsat = np.array([r["verdict"] == "unsat" for r in recs])
    gn = np.array([r["nodes"] for r in recs])
    cert = H._engine_cert_refutes(fb)
    unc = unsat & ~cert & (gn > 0)
    enum = unc & (out["nodes"] == 0)
    print(f"{name}: {len(recs)} records, {int(unsat.sum())} Unsat, {int(unc.sum())} searched by the reference "
          f"without a certificate, {int(enum.sum())} of them decided by enumeration")
