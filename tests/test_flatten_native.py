"""Native query emission (csrc/flatten_native.cpp)
against the interpreted restatement of the wire format (wire.flatten_py):
identical arrays, names and errors, on every golden set, on the reference's
own term objects, and on the edge cases of the name-resolution rules
(solver.py:372-374)."""
from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import GOLDEN_SETS, REF_SRC, load_golden, reference_available

from paper_2601_21552_b200 import terms, wire
from paper_2601_21552_b200.solver import BinE, Constraint, Lit, SolverVar, VarRef

FIELDS = ("var_begin", "var_lo", "var_hi", "con_begin", "con_rel", "con_lhs", "con_rhs",
          "node_begin", "node_op", "node_a", "node_b", "lit_begin", "lits")


def same(a, b):
    for k in FIELDS:
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y), k
    assert a.var_names == b.var_names


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_native_equals_python_on_golden_sets(name):
    recs = load_golden(name)
    same(wire.flatten(recs), wire.flatten_py(recs))
    objs = [terms.query_from_json(r) for r in recs]
    same(wire.flatten(objs), wire.flatten_py(objs))


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_native_on_reference_objects():
    sys.path.insert(0, str(REF_SRC))
    import scuba_mini.solver as R
    recs = load_golden("corpus_m1048576") + load_golden("random_solver")
    objs = [terms.query_from_json(r, types=R) for r in recs]
    assert type(objs[0][1][0]).__module__ == "scuba_mini.solver"
    same(wire.flatten(objs), wire.flatten_py(objs))


x, y = VarRef("x"), VarRef("y")


def q(vars_, cons):
    return ([SolverVar(*v) for v in vars_], cons)


EDGE = [
    q([("x", 0, 9), ("y", 0, 9), ("x", 2, 5)], [Constraint("<", x, y)]),          # last decl wins
    q([("x", 3, 1), ("y", 0, 9), ("z", 5, 2)], [Constraint("=", x, Lit(1))]),      # empty domain -> slot 0
    q([("x", 0, 9)], [Constraint("=", BinE("+", x, x), BinE("+", x, x))]),         # hash-consing
    q([("x", -(1 << 100), 1 << 100)], [Constraint(">=", x, Lit(-(1 << 126)))]),   # wide values
    q([("x", 0, 9)], []),
    ([], []),
]


def test_native_edge_cases():
    same(wire.flatten(EDGE), wire.flatten_py(EDGE))


@pytest.mark.parametrize("bad,exc", [
    (q([("x", 0, 9)], [Constraint("<", x, y)]), KeyError),
    (q([("x", 0, 9)], [Constraint("!=", x, Lit(1))]), ValueError),
    (q([("x", 0, 9)], [Constraint("<", BinE("^", x, x), Lit(1))]), ValueError),
    (q([("x", 0, 9)], [Constraint("<", True, Lit(1))]), ValueError),
    (q([("x", 0, 1 << 130)], [Constraint("<", x, Lit(1))]), OverflowError),
    (q([("x", 0, 9)], [Constraint("<", x, Lit(1 << 127))]), OverflowError),
])
def test_native_errors_match(bad, exc):
    for fn in (wire.flatten, wire.flatten_py):
        with pytest.raises(exc) as e:
            fn([bad])
        if exc is KeyError:
            assert e.value.args == ("y",)


@pytest.mark.parametrize("case", [
    # an out-of-range bound overwritten by a later declaration is not stored
    [q([("x", 0, 1 << 130), ("y", 0, 1), ("x", 0, 9)], [Constraint("<", x, y)])],
    # an out-of-range empty declaration is stored into slot 0 (then overflows)
    [q([("x", 0, 9), ("y", 1 << 130, 0)], [Constraint("<", x, y)])],
    [q([("x", 0, 9), ("y", 5, -(1 << 130))], [Constraint("<", x, y)])],
])
def test_native_range_check_follows_stored_values(case):
    def outcome(fn):
        try:
            fb = fn(case)
            return ("ok", fb.var_lo.tolist(), fb.var_hi.tolist())
        except OverflowError as e:
            return ("overflow", str(e))
    assert outcome(wire.flatten) == outcome(wire.flatten_py)
