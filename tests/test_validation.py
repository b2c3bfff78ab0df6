"""Batch validation in the C ABI (host.cpp validate / validate_offsets /
validate_terms): a malformed query is reported with the lowest offending
index and the same message whichever path its compile takes -- a structure
seen before (the structure cache skips re-checking terms equal to an already
validated query's, so a corrupted copy must miss it), a new one, a query with
an empty domain (decided before the cache), a non-literal divisor (never
cached).  CPU only: oob_host_bench runs the host pipeline without a device."""
from __future__ import annotations

import copy

import numpy as np
import pytest

from paper_2601_21552_b200 import _lib
from paper_2601_21552_b200.wire import flatten


def _q(lo=0, hi=7, div_var=False):
    d = "y" if div_var else 3
    return {"vars": [["x", lo, hi], ["y", 1, 5]],
            "cons": [["<", ["+", "x", 2], ["/", "y", d]], ["=", "x", 1]]}


def _batch(n=6, **kw):
    return flatten([_q(**kw) for _ in range(n)])


def _fail(fb):
    with pytest.raises(ValueError) as e:
        _lib.host_bench(fb, flags=_lib.F_FAST)
    return str(e.value)


def test_valid_batch_passes():
    _lib.host_bench(_batch(), flags=_lib.F_FAST)
    _lib.host_bench(_batch(div_var=True), flags=_lib.F_FAST)


@pytest.mark.parametrize("kw", [{}, {"div_var": True}, {"lo": 9, "hi": 2}])
def test_corrupted_terms_are_reported_on_every_path(kw):
    for field, value, msg in (("node_op", 9, "unknown operator code 9"),
                              ("node_a", 99, None),
                              ("con_rel", 7, "unknown relation code 7"),
                              ("con_lhs", 99, "constraint root out of range")):
        fb = _batch(**kw)
        _lib.host_bench(fb, flags=_lib.F_FAST)  # the valid structure is cached first
        bad = copy.deepcopy(fb)
        q = 4
        base = {"node_op": bad.node_begin, "node_a": bad.node_begin, "con_rel": bad.con_begin,
                "con_lhs": bad.con_begin}[field][q]
        getattr(bad, field)[base] = value
        text = _fail(bad)
        assert f"query {q}:" in text, text
        if msg:
            assert msg in text, text


def test_operand_order_and_divisor_index_checked():
    fb = _batch()
    _lib.host_bench(fb, flags=_lib.F_FAST)
    bad = copy.deepcopy(fb)
    q = 3
    nb0, nb1 = int(bad.node_begin[q]), int(bad.node_begin[q + 1])
    ops = bad.node_op[nb0:nb1]
    i = int(np.nonzero(ops == 5)[0][0])  # the "/" node: its divisor after it
    bad.node_b[nb0 + i] = nb1 - nb0 - 1 if i < nb1 - nb0 - 1 else i
    text = _fail(bad)
    assert "query 3:" in text and "operand node not before its parent" in text, text


def test_decreasing_offsets_and_lowest_index():
    fb = _batch()
    bad = copy.deepcopy(fb)
    bad.con_begin[5] = bad.con_begin[4] - 1
    assert "decreasing offsets" in _fail(bad)
    bad = copy.deepcopy(fb)
    for q in (2, 4):
        bad.node_op[bad.node_begin[q]] = 9
    assert "query 2:" in _fail(bad)
