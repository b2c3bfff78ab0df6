"""B200-native engine for the per-access OOB satisfiability check of
arXiv 2601.21552 (reference: "scuba-mini", pure Python).

Public surface mirrors `scuba_mini.solver` (see `solver.py`); the analyzer
integration lives in `analyzer.py`; the C ABI in include/scuba_oob.h.
"""
from .solver import (  # noqa: F401
    BinE,
    Constraint,
    Lit,
    Sat,
    SolverVar,
    Timeout,
    Unsat,
    VarRef,
    check_model,
    divisor_side_constraints,
    propagate,
    solve,
    solve_batch,
    tdiv,
    tmod,
)

__version__ = "0.1.0"
