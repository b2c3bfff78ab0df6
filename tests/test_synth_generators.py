"""The seeded generator built into oracle/ (bench.py's reference arm) emits
byte-identical batches to the engine library's copy."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2601_21552_b200 import synth

FIELDS = ("var_begin", "var_lo", "var_hi", "con_begin", "con_rel", "con_lhs", "con_rhs",
          "node_begin", "node_op", "node_a", "node_b", "lit_begin", "lits")


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5", "c5s"])
def test_oracle_side_generator_identical(cfg):
    a = synth.generate(cfg, 3000, first=777, names=False)
    b = oracle.synth_generate(cfg, 3000, first=777)
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.tmpl, b.tmpl)
