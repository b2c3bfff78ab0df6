"""Term and verdict types of the bounded-integer OOB query, plus its JSON form.

These mirror the value types the reference solver exchanges with its callers
(`/root/reference/pkg/src/scuba_mini/solver.py:32-84`): terms `Lit`, `VarRef`,
`BinE`; `Constraint`; `SolverVar`; verdicts `Sat`, `Unsat`, `Timeout`.  They
exist so the engine can be used (and tested on the GPU box) without the
reference package.  When the reference package is importable, its own objects
are accepted everywhere these are (the flattener reads attributes, not
classes), and `install()` returns the reference's verdict classes.

JSON form (used by the golden fixtures and the CLI tools):
  term        int              -> Lit(value)
              str              -> VarRef(name)
              [op, l, r]       -> BinE(op, l, r)      op in + - * / %
  constraint  [rel, lhs, rhs]  rel in < <= = >= >
  variable    [name, lo, hi]
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Union

RELS = ("<", "<=", "=", ">=", ">")  # solver.py:26
OPS = ("+", "-", "*", "/", "%")     # solver.py:44


@dataclass(frozen=True)
class Lit:
    value: int


@dataclass(frozen=True)
class VarRef:
    name: str


@dataclass(frozen=True)
class BinE:
    op: str
    left: "SExpr"
    right: "SExpr"


SExpr = Union[Lit, VarRef, BinE]


@dataclass(frozen=True)
class Constraint:
    rel: str
    lhs: SExpr
    rhs: SExpr


@dataclass(frozen=True)
class SolverVar:
    name: str
    lo: int
    hi: int


@dataclass
class Sat:
    model: dict


@dataclass
class Unsat:
    pass


@dataclass
class Timeout:
    elapsed: float


Verdict = Union[Sat, Unsat, Timeout]


# ----- JSON form ------------------------------------------------------------


def term_to_json(e):
    """Encode a term (ours or the reference's) in the compact JSON form."""
    if hasattr(e, "op"):
        return [e.op, term_to_json(e.left), term_to_json(e.right)]
    if hasattr(e, "value"):
        return int(e.value)
    return str(e.name)


def term_from_json(j, lit=Lit, var=VarRef, bine=BinE):
    if isinstance(j, bool):
        raise ValueError("boolean is not a term")
    if isinstance(j, int):
        return lit(j)
    if isinstance(j, str):
        return var(j)
    op, l, r = j
    return bine(op, term_from_json(l, lit, var, bine),
                term_from_json(r, lit, var, bine))


def query_to_json(variables, constraints) -> dict:
    return {
        "vars": [[v.name, int(v.lo), int(v.hi)] for v in variables],
        "cons": [[c.rel, term_to_json(c.lhs), term_to_json(c.rhs)]
                 for c in constraints],
    }


def query_from_json(q: dict, types=None):
    """(variables, constraints) from the JSON form, built from `types`
    (a module or namespace exposing Lit/VarRef/BinE/Constraint/SolverVar;
    default: this module)."""
    t = types
    lit = getattr(t, "Lit", Lit)
    var = getattr(t, "VarRef", VarRef)
    bine = getattr(t, "BinE", BinE)
    con = getattr(t, "Constraint", Constraint)
    svar = getattr(t, "SolverVar", SolverVar)
    variables = [svar(n, int(lo), int(hi)) for n, lo, hi in q["vars"]]
    constraints = [
        con(rel, term_from_json(l, lit, var, bine),
            term_from_json(r, lit, var, bine))
        for rel, l, r in q["cons"]
    ]
    return variables, constraints


def verdict_to_json(v) -> dict:
    name = type(v).__name__
    if name == "Sat":
        return {"verdict": "sat", "model": {k: int(x) for k, x in v.model.items()}}
    if name == "Unsat":
        return {"verdict": "unsat"}
    if name == "Timeout":
        return {"verdict": "timeout"}
    raise TypeError(f"not a verdict: {v!r}")
