"""Flat wire format: round trips, int128 words, the reference's dict/list
semantics for variables, and error conventions."""
from __future__ import annotations

import pytest

from conftest import GOLDEN_SETS, load_golden

from paper_2601_21552_b200 import terms
from paper_2601_21552_b200.wire import flatten, join128, split128, words_to_ints


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_json_round_trip(name):
    recs = load_golden(name)
    fb = flatten(recs)
    assert fb.n == len(recs)
    for q, r in enumerate(recs):
        j = fb.query_json(q)
        assert j["vars"] == r["vars"] and j["cons"] == r["cons"]


def test_objects_and_json_flatten_identically():
    recs = load_golden("random_accept")[:50]
    objs = [terms.query_from_json(r) for r in recs]
    a, b = flatten(recs), flatten(objs)
    for f in ("var_begin", "var_lo", "con_rel", "con_lhs", "node_op", "node_a", "node_b", "lits"):
        assert (getattr(a, f) == getattr(b, f)).all(), f


@pytest.mark.parametrize("v", [0, 1, -1, 2**63, -(2**63), 2**64 + 5, -(2**100) - 7, 2**127 - 1, -(2**127)])
def test_int128_words(v):
    lo, hi = split128(v)
    assert join128(lo, hi) == v


def test_out_of_range_literal_raises():
    with pytest.raises(OverflowError):
        flatten([{"vars": [["x", 0, 1]], "cons": [["<", "x", 2**130]]}])


def test_hash_consing_shares_structure():
    fb = flatten([{"vars": [["x", 0, 9], ["y", 0, 9]],
                   "cons": [["=", ["/", "x", ["+", "y", 1]], 2], ["<", ["+", "y", 1], 5]]}])
    # x, y, 1, (+ y 1), (/ x (+ y 1)), 2, 5: the repeated (+ y 1) is one node
    assert int(fb.node_begin[1]) == 7
    assert words_to_ints(fb.lits) == [1, 2, 5]


def test_duplicate_names_follow_dict_semantics():
    fb = flatten([{"vars": [["x", 0, 9], ["y", 0, 3], ["x", 2, 4]], "cons": []}])
    assert fb.names(0) == ["x", "y"]
    assert words_to_ints(fb.var_lo) == [2, 0] and words_to_ints(fb.var_hi) == [4, 3]


def test_undeclared_variable_and_unknown_op():
    with pytest.raises(KeyError):
        flatten([{"vars": [["x", 0, 1]], "cons": [["<", "z", 2]]}])
    with pytest.raises(ValueError):
        flatten([{"vars": [["x", 0, 1]], "cons": [["<", ["^", "x", 1], 2]]}])
    with pytest.raises(ValueError):
        flatten([{"vars": [["x", 0, 1]], "cons": [["!=", "x", 1]]}])


def test_empty_domain_query_is_unsat_without_resolving_terms():
    """solver.py:374: any lo > hi is Unsat before the constraints are touched,
    so an undeclared variable or unknown operator there raises nothing."""
    from paper_2601_21552_b200.wire import flatten_py
    from paper_2601_21552_b200.wire import flatten as flatten_any
    q = {"vars": [["x", 0, 5], ["y", 3, 1]],
         "cons": [["<", "undeclared", 3], ["=", ["^", "x", 2], 1]]}
    for fl in (flatten_py, flatten_any):
        fb = fl([q])
        assert fb.n == 1 and int(fb.con_begin[1]) == 0
