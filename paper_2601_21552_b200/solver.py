"""Drop-in for `scuba_mini.solver` backed by the B200 engine.

Same names, argument meaning and error behaviour as the reference module
(/root/reference/pkg/src/scuba_mini/solver.py):

  solve(variables, constraints, timeout_s=30.0) -> Sat | Unsat | Timeout   (:363)
  propagate(domains, constraints, deadline=None) -> dict | None           (:264)
  check_model(constraints, model) -> bool                                 (:319)
  divisor_side_constraints(constraints) -> list[Constraint]               (:345)
  tdiv(a, b), tmod(a, b)                                                  (:94-102)

plus the batched form the analyzer integration uses:

  solve_batch(queries, timeout_s=30.0, ...) -> list[Verdict]

Decisions run on the GPU through the C ABI (include/scuba_oob.h); there is no
CPU fallback.  Verdicts are the reference's, including the first model of the
reference DFS (same traversal, same 10**18 clamp, same 10 000-pass cap).
Terms may be this package's types or the reference's own objects.
"""
from __future__ import annotations

import time
from typing import Iterable, Optional

import numpy as np

from . import _lib
from .terms import (  # noqa: F401  (re-exported API)
    RELS,
    BinE,
    Constraint,
    Lit,
    Sat,
    SolverVar,
    Timeout,
    Unsat,
    VarRef,
    Verdict,
)
from .wire import FlatBatch, flatten, split128, words_to_ints

_INF = 10**18
_PASS_CAP = 10_000

DEFAULT_VERDICT_TYPES = (Sat, Unsat, Timeout)


# ----- C-truncating integer helpers (solver.py:94-102) -----------------------

def tdiv(a: int, b: int) -> int:
    """Truncating division, rounding toward zero like C's ``/``."""
    q = abs(a) // abs(b)
    return q if (a < 0) == (b < 0) else -q


def tmod(a: int, b: int) -> int:
    """C remainder ``a - b * tdiv(a, b)``; the sign follows ``a``."""
    return a - b * tdiv(a, b)


# ----- side constraints (solver.py:334-357) ----------------------------------

def _is_lit(e) -> bool:
    return not hasattr(e, "op") and hasattr(e, "value")


def divisor_side_constraints(constraints):
    """``divisor >= 1`` for each distinct non-literal divisor, in pre-order of
    the constraint list (left side before right side).  Built from the same
    classes as the input constraints."""
    found = []

    def walk(e):
        if not hasattr(e, "op"):
            return
        if e.op in ("/", "%") and not (_is_lit(e.right) and e.right.value >= 1):
            if e.right not in found:
                found.append(e.right)
        walk(e.left)
        walk(e.right)

    con_cls = Constraint
    lit_cls = Lit
    for c in constraints:
        con_cls = type(c)
        walk(c.lhs)
        walk(c.rhs)
        for side in (c.lhs, c.rhs):
            if _is_lit(side):
                lit_cls = type(side)
    return [con_cls(">=", d, lit_cls(1)) for d in found if not _is_lit(d)]


# ----- batched decision --------------------------------------------------------

def _verdicts_from(out, fb: FlatBatch, types, raise_errors=True):
    SatT, UnsatT, TimeoutT = types
    verdicts = []
    model = out["model"]
    errors = []
    for q in range(fb.n):
        v = int(out["verdict"][q])
        if v == _lib.SAT:
            vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q + 1])
            vals = words_to_ints(model[vb:ve])
            verdicts.append(SatT(dict(zip(fb.names(q), vals))))
        elif v == _lib.UNSAT:
            verdicts.append(UnsatT())
        elif v == _lib.TIMEOUT:
            verdicts.append(TimeoutT(max(float(out["elapsed"][q]), 1e-9)))
        else:
            verdicts.append(None)
            errors.append(q)
    if errors and raise_errors:
        raise _lib.EngineError(
            f"{len(errors)} of {fb.n} queries could not be decided exactly on the "
            f"GPU: {out['error'] or 'error verdict'}")
    return verdicts


def solve_flat(fb: FlatBatch, timeout_s: float = 30.0, *, node_budget: int = 0,
               n_gpus: int = 0, device: int = 0, flags: int = 0, heavy_nodes: int = 0,
               jit_min: int = 0) -> dict:
    """Decide a FlatBatch; returns raw numpy results (verdict codes, model
    words, nodes, passes, elapsed).  Raises on engine errors.  heavy_nodes:
    DFS nodes after which a query moves to the warp-cooperative frontier
    kernel (0 = default, < 0 = never)."""
    out = _lib.solve_flat(fb, timeout_s, node_budget, n_gpus, device, flags, heavy_nodes, jit_min)
    rc = out["status"]
    if rc == _lib.OOB_E_INVALID:
        raise ValueError(out["error"])
    if rc not in (_lib.OOB_OK, _lib.OOB_E_RANGE):
        raise _lib.EngineError(f"oob_solve_batch failed (status {rc}): {out['error']}")
    return out


MODES = {"canonical": 0, "fast": _lib.F_FAST}


def solve_batch(queries: Iterable, timeout_s: float = 30.0, *, node_budget: int = 0,
                n_gpus: int = 0, device: int = 0, verdict_types=None,
                stats: bool = False, mode: str = "canonical"):
    """Decide many queries in one GPU batch.

    `queries`: iterable of `(variables, constraints)` pairs (reference-shaped
    objects or the JSON form).  Returns the list of verdicts in input order
    (and the raw result arrays when `stats`).  `mode`: "canonical" (exact
    emulation of the reference search: verdicts, models and node/pass
    counters are the reference's) or "fast" (heavy queries first meet the
    symbolic Unsat prover: verdicts and Sat models are the reference's,
    counters of refuted queries are 0)."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r} (canonical, fast)")
    fb = flatten(list(queries))
    out = solve_flat(fb, timeout_s, node_budget=node_budget, n_gpus=n_gpus, device=device,
                     flags=MODES[mode])
    verdicts = _verdicts_from(out, fb, verdict_types or DEFAULT_VERDICT_TYPES)
    return (verdicts, out) if stats else verdicts


def solve(variables, constraints, timeout_s: float = 30.0, *, mode: str = "canonical"):
    """Decide the conjunction over the given finite domains (solver.py:363).
    One query runs on one device (n_gpus=1)."""
    types = DEFAULT_VERDICT_TYPES
    return solve_batch([(variables, constraints)], timeout_s, n_gpus=1, verdict_types=types, mode=mode)[0]


# ----- propagate / check_model ------------------------------------------------

class Deadline(Exception):
    """Raised by propagate() when its deadline has already passed (the
    reference raises its private _Deadline, solver.py:272-273)."""


def propagate(domains: dict, constraints, deadline: Optional[float] = None):
    """Narrow ``domains`` to a propagation fixpoint; None on contradiction."""
    if deadline is not None and time.monotonic() > deadline:
        raise Deadline()
    names = list(domains)
    variables = [(n, int(domains[n][0]), int(domains[n][1])) for n in names]
    fb = _flatten_raw(variables, constraints)
    lo, hi, st = _lib.propagate_flat(fb)
    if int(st[0]) == 0:
        return None
    los = words_to_ints(lo[: len(names)])
    his = words_to_ints(hi[: len(names)])
    return {n: (a, b) for n, a, b in zip(names, los, his)}


def check_model(constraints, model: dict) -> bool:
    """Exact evaluation of the conjunction under a complete assignment."""
    names = list(model)
    variables = [(n, int(model[n]), int(model[n])) for n in names]
    fb = _flatten_raw(variables, constraints)
    words = np.zeros((max(len(names), 1), 2), dtype=np.int64)
    for i, n in enumerate(names):
        words[i] = split128(int(model[n]))
    return bool(_lib.check_model_flat(fb, words)[0])


def _flatten_raw(variables, constraints) -> FlatBatch:
    """Like flatten() but keeps empty domains as given (propagate's input is a
    plain dict and may legitimately hold lo > hi entries)."""
    fb = flatten([(variables, constraints)])
    vb = 0
    for i, (_, a, b) in enumerate(variables):
        fb.var_lo[vb + i] = split128(a)
        fb.var_hi[vb + i] = split128(b)
    return fb
