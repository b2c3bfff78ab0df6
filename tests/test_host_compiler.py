"""Host compiler on CPU (no device): exact-regime classification, the
per-thread structure cache, and the run-time specialisation source."""
from __future__ import annotations

import numpy as np

from paper_2601_21552_b200 import _lib, synth
from paper_2601_21552_b200.wire import flatten


def test_regimes_of_the_synthetic_streams():
    # wide regimes come from products of 2^31 / 2^59 declared domains
    r3 = _lib.query_regime(synth.generate("c3", 4000, names=False))
    r4 = _lib.query_regime(synth.generate("c4", 4000, names=False))
    assert set(np.unique(r3)) <= {1, 2, 3} and (r3 == 1).mean() > 0.6
    assert (r4 >= 2).mean() > 0.3


def test_regime_is_per_query_not_per_structure():
    # identical structure, different domains: the bound proof is per query
    small = {"vars": [["x", 0, 10], ["y", 0, 10]], "cons": [["<", ["*", "x", "y"], 50]]}
    big = {"vars": [["x", 0, 2**40], ["y", 0, 2**40]], "cons": [["<", ["*", "x", "y"], 50]]}
    huge = {"vars": [["x", 0, 2**100], ["y", 0, 2**100]], "cons": [["<", ["*", "x", "y"], 50]]}
    r = _lib.query_regime(flatten([small, big, huge, small]))
    assert list(r) == [1, 2, 3, 1]


def test_structure_cache_keeps_side_constraints_exact():
    # the same terms with a literal divisor and with a variable divisor:
    # only the second gets the divisor side constraint (solver.py:345-357)
    lit = {"vars": [["x", 0, 9], ["d", 1, 3]], "cons": [["<", ["/", "x", 3], 2]]}
    var = {"vars": [["x", 0, 9], ["d", 1, 3]], "cons": [["<", ["/", "x", "d"], 2]]}
    fb = flatten([lit, var, lit])
    s0, _ = _lib.jit_compile(fb, 0)
    s1, _ = _lib.jit_compile(fb, 1)
    s2, _ = _lib.jit_compile(fb, 2)
    assert s0 == s2
    assert s0.count("bool prop") == 1 and s1.count("bool prop") == 2


def test_host_pipeline_runs_without_a_device():
    fb = synth.generate("c3", 20000, names=False)
    ms = _lib.host_bench(fb)
    assert ms.shape == (3,) and (ms > 0).all()
